// inst_keycorridor.cu — kernel instantiations of one family group (compiled in
// parallel with the other groups; see step_kernel.cuh).
#include "step_kernel.cuh"

namespace navix {

cudaError_t launch_group_keycorridor(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s, bool* handled) {
  *handled = true;
  switch (key) {
    case FAM_KEYCORRIDOR * 10000 + 307: return launch_fhw<FAM_KEYCORRIDOR, 3, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 507: return launch_fhw<FAM_KEYCORRIDOR, 5, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 707: return launch_fhw<FAM_KEYCORRIDOR, 7, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 1010: return launch_fhw<FAM_KEYCORRIDOR, 10, 10>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 1313: return launch_fhw<FAM_KEYCORRIDOR, 13, 13>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 1616: return launch_fhw<FAM_KEYCORRIDOR, 16, 16>(mode, a, n_tiles, s);
    default: *handled = false; return cudaSuccess;
  }
}

}  // namespace navix
