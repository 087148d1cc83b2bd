// Throughput instantiation: fp32 deviation storage (152 B per cell update).
#define FSG_PREC 32
#include "fsg_kernels.cuh"
namespace fsg {
const Launchers& launchers_fp32() { return p32::kLaunchers; }
}  // namespace fsg

#ifdef FSG_TIMING
// dev build only (libfsg_dbg.so): copy out and re-arm the phase timeline ring
extern "C" int fsg_debug_timeline(unsigned long long* out) {
  static unsigned long long init[64 * fsg::TL_SLOTS];
  for (int i = 0; i < 64 * fsg::TL_SLOTS; ++i) init[i] = (i & 1) ? 0ull : ~0ull;
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, fsg::g_tl, sizeof init);
  return (int)cudaMemcpyToSymbol(fsg::g_tl, init, sizeof init);
}
#endif

#ifdef FSG_TIMING
extern "C" int fsg_debug_blocks(unsigned long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, fsg::g_blk, sizeof(unsigned long long) * 8192 * 4);
}
#endif

#ifdef FSG_TIMING
extern "C" int fsg_debug_mkt(unsigned long long* out) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, fsg::g_mkt, sizeof(unsigned long long) * 4096 * 16);
}
#endif
