// dispatch.cu — host-side dispatch of the step kernels (one family group per
// translation unit, inst_*.cu) and the two small utility kernels.
#include <cstdint>
#include <mutex>

#include "layout.h"
#include "philox.cuh"

namespace navix {

// One family group's instantiations (inst_*.cu): launches the kernel for
// dispatch key `key` (family * 10000 + H * 100 + W) and sets *handled, or
// leaves *handled false if the key is not in the group.
using GroupLauncher = cudaError_t (*)(int key, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s,
                                      bool* handled);
cudaError_t launch_group_empty(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);
cudaError_t launch_group_doorkey(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);
cudaError_t launch_group_dynobs(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);
cudaError_t launch_group_keycorridor(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);
cudaError_t launch_group_lava_crossing_distshift(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);
cudaError_t launch_group_gotodoor_fourrooms(int, int, const KernelArgs&, int64_t, cudaStream_t, bool*);

// SM count of the current device (cached per device): grid-stride utility
// kernels launch a few waves' worth of CTAs, not a hard-coded 148.
int current_device_sm_count() {
  constexpr int MAXD = 64;
  static std::once_flag once[MAXD];
  static int n_sm[MAXD];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAXD) return 148;
  std::call_once(once[dev], [dev] {
    if (cudaDeviceGetAttribute(&n_sm[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n_sm[dev] < 1)
      n_sm[dev] = 148;
  });
  return n_sm[dev];
}

// ------------------------------------------------------------------ other kernels
__global__ void sample_actions_kernel(uint8_t* out, int64_t n, int64_t steps, uint32_t env_begin, uint32_t t0,
                                      uint32_t klo, uint32_t khi, uint32_t n_actions) {
  const int64_t total = n * steps;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / n, env = i % n;
    const uint4 w = philox4x32_10(make_uint4(env_begin + (uint32_t)env, t0 + (uint32_t)t, 2u << 16, 0u), klo, khi);
    out[i] = (uint8_t)bounded(w.x, n_actions);
  }
}

__global__ void stats_reduce_kernel(const unsigned long long* slots, long long* out8) {
  __shared__ unsigned long long part[8][32];
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;  // 256 threads: 8 counters x 32 lanes
  unsigned long long s = 0;
  for (int i = lane; i < NSLOT; i += 32) s += slots[(size_t)i * 8 + k];
  part[k][lane] = s;
  __syncthreads();
  if (lane == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < 32; ++i) t += part[k][i];
    out8[k] = (long long)t;
  }
}

// GoToDoor's mission (Table 6 `on_door_done`, "the colour specified in the
// mission"): the colour of each env's target door, read from the agent
// record (byte 7 = (x << 4) | y) and the HBM grid.  out[e] in 0..5.
__global__ void mission_kernel(const uint64_t* grid, const uint64_t* agent, int64_t n, int rw, int h,
                               uint8_t* out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e / TILE, slot = tile * TILE + slot_of_env((int)(e % TILE));
    const uint32_t t = (uint32_t)(agent[slot] >> 56);
    const int x = (int)(t >> 4), y = (int)(t & 15);
    const uint64_t plane = grid[(tile * h * rw + y * rw + (x >> 3)) * TILE + (slot - tile * TILE)];
    out[e] = (uint8_t)((plane >> (8 * (x & 7) + 4)) & 7);
  }
}

cudaError_t launch_mission(const uint64_t* grid, const uint64_t* agent, int64_t n, int rw, int h, uint8_t* out,
                           cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  const int64_t cap = (int64_t)current_device_sm_count() * 16;
  if (blocks > cap) blocks = cap;
  mission_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(grid, agent, n, rw, h, out);
  return cudaPeekAtLastError();
}

cudaError_t launch_env_kernel(const EnvConfig& c, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s) {
  static const GroupLauncher groups[] = {launch_group_empty, launch_group_doorkey, launch_group_dynobs, launch_group_keycorridor, launch_group_lava_crossing_distshift, launch_group_gotodoor_fourrooms};
  const int key = c.family * 10000 + c.height * 100 + c.width;
  for (GroupLauncher g : groups) {
    bool handled = false;
    const cudaError_t e = g(key, mode, a, n_tiles, s, &handled);
    if (handled) return e;
  }
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_sample_actions(uint8_t* out, int64_t n, int64_t steps, uint32_t env_begin, uint32_t t0,
                                  uint64_t seed, uint32_t n_actions, cudaStream_t s) {
  const int64_t total = n * steps;
  int64_t blocks = (total + 255) / 256;
  const int64_t cap = (int64_t)current_device_sm_count() * 64;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  sample_actions_kernel<<<(unsigned)blocks, 256, 0, s>>>(out, n, steps, env_begin, t0, (uint32_t)seed,
                                                         (uint32_t)(seed >> 32), n_actions);
  return cudaPeekAtLastError();
}

cudaError_t launch_stats_reduce(const unsigned long long* slots, long long* out8, cudaStream_t s) {
  stats_reduce_kernel<<<1, 256, 0, s>>>(slots, out8);
  return cudaPeekAtLastError();
}

}  // namespace navix
