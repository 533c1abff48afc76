// inst_doorkey.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_doorkey(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_DOORKEY * 10000 + 505: return launch_fhw<FAM_DOORKEY, 5, 5>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 606: return launch_fhw<FAM_DOORKEY, 6, 6>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 808: return launch_fhw<FAM_DOORKEY, 8, 8>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 1616: return launch_fhw<FAM_DOORKEY, 16, 16>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
