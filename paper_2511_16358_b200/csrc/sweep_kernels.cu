// sweep_kernels.cu — the float instances of the persistent whole-sweep kernel (sweep.cuh),
// one per lane mapping, plus the dispatcher; the double instances are in
// sweep_kernels_f64.cu.  Separate translation units so that they compile in parallel with
// ifctn.cu (build.py).
#include "sweep.cuh"

namespace ifctn {

const void* persistent_kernel_f64(int epl, int lpf);

const void* persistent_kernel(int esize, int epl, int lpf) {
    if (esize != 4) return persistent_kernel_f64(epl, lpf);
    if (epl == 4) return lpf == 16 ? (const void*)sweep_persistent<float, 4, 16> : (const void*)sweep_persistent<float, 4, 32>;
    if (epl == 8) return (const void*)sweep_persistent<float, 8, 32>;
    return (const void*)sweep_persistent<float, 16, 32>;
}

}  // namespace ifctn
