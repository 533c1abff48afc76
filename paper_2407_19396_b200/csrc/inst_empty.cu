// inst_empty.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_empty(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_EMPTY * 10000 + 505: return launch_fhw<FAM_EMPTY, 5, 5>(mode, a, n_tiles, s);
    case FAM_EMPTY * 10000 + 606: return launch_fhw<FAM_EMPTY, 6, 6>(mode, a, n_tiles, s);
    case FAM_EMPTY * 10000 + 808: return launch_fhw<FAM_EMPTY, 8, 8>(mode, a, n_tiles, s);
    case FAM_EMPTY * 10000 + 1616: return launch_fhw<FAM_EMPTY, 16, 16>(mode, a, n_tiles, s);
    case FAM_EMPTY_RANDOM * 10000 + 505: return launch_fhw<FAM_EMPTY_RANDOM, 5, 5>(mode, a, n_tiles, s);
    case FAM_EMPTY_RANDOM * 10000 + 606: return launch_fhw<FAM_EMPTY_RANDOM, 6, 6>(mode, a, n_tiles, s);
    case FAM_EMPTY_RANDOM * 10000 + 808: return launch_fhw<FAM_EMPTY_RANDOM, 8, 8>(mode, a, n_tiles, s);
    case FAM_EMPTY_RANDOM * 10000 + 1616: return launch_fhw<FAM_EMPTY_RANDOM, 16, 16>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
