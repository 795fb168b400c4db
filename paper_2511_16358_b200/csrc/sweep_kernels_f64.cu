// sweep_kernels_f64.cu — the double instances of the persistent whole-sweep kernel
// (sweep.cuh); see sweep_kernels.cu.
#include "sweep.cuh"

namespace ifctn {

const void* persistent_kernel_f64(int epl, int lpf) {
    if (epl == 2) return lpf == 16 ? (const void*)sweep_persistent<double, 2, 16> : (const void*)sweep_persistent<double, 2, 32>;
    if (epl == 4) return (const void*)sweep_persistent<double, 4, 32>;
    return (const void*)sweep_persistent<double, 8, 32>;
}

}  // namespace ifctn
