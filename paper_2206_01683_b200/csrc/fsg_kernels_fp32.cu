// Throughput instantiation: fp32 deviation storage (152 B per cell update).
#define FSG_PREC 32
#include "fsg_kernels.cuh"
namespace fsg {
const Launchers& launchers_fp32() { return p32::kLaunchers; }
}  // namespace fsg
