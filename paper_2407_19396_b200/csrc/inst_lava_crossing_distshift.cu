// inst_lava_crossing_distshift.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_lava_crossing_distshift(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_LAVAGAP * 10000 + 505: return launch_fhw<FAM_LAVAGAP, 5, 5>(mode, a, n_tiles, s);
    case FAM_LAVAGAP * 10000 + 606: return launch_fhw<FAM_LAVAGAP, 6, 6>(mode, a, n_tiles, s);
    case FAM_LAVAGAP * 10000 + 707: return launch_fhw<FAM_LAVAGAP, 7, 7>(mode, a, n_tiles, s);
    case FAM_DISTSHIFT1 * 10000 + 709: return launch_fhw<FAM_DISTSHIFT1, 7, 9>(mode, a, n_tiles, s);
    case FAM_DISTSHIFT2 * 10000 + 709: return launch_fhw<FAM_DISTSHIFT2, 7, 9>(mode, a, n_tiles, s);
    case FAM_CROSSING * 10000 + 909: return launch_fhw<FAM_CROSSING, 9, 9>(mode, a, n_tiles, s);
    case FAM_CROSSING * 10000 + 1111: return launch_fhw<FAM_CROSSING, 11, 11>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
