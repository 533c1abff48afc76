// inst_gotodoor_fourrooms.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_gotodoor_fourrooms(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_FOURROOMS * 10000 + 1717: return launch_fhw<FAM_FOURROOMS, 17, 17>(mode, a, n_tiles, s);
    case FAM_GOTODOOR * 10000 + 505: return launch_fhw<FAM_GOTODOOR, 5, 5>(mode, a, n_tiles, s);
    case FAM_GOTODOOR * 10000 + 606: return launch_fhw<FAM_GOTODOOR, 6, 6>(mode, a, n_tiles, s);
    case FAM_GOTODOOR * 10000 + 808: return launch_fhw<FAM_GOTODOOR, 8, 8>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
