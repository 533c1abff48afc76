// inst_dynobs.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_dynobs(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_DYNOBS * 10000 + 505: return launch_fhw<FAM_DYNOBS, 5, 5>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 606: return launch_fhw<FAM_DYNOBS, 6, 6>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 808: return launch_fhw<FAM_DYNOBS, 8, 8>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 1616: return launch_fhw<FAM_DYNOBS, 16, 16>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
