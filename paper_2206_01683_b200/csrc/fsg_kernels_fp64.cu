// Parity instantiation: fp64 storage, the reference's operation order.
// Built with --fmad=false (no FMA contraction) so that every rounding step
// matches the reference's x86-64 fp64 evaluation bit-for-bit.
#define FSG_PREC 64
#include "fsg_kernels.cuh"
namespace fsg {
const Launchers& launchers_fp64() { return p64::kLaunchers; }
}  // namespace fsg
