// tools/sol_mix.cu — speed-of-light probe for the step kernel's memory traffic.
//
// Moves exactly the bytes of one DoorKey-8x8 env-step with the product's
// layouts and store path, but no environment logic: per env read 64 B of grid
// rows (u64 [tile][8][128]), an 8 B agent record and a 1 B action; write the
// 8 B agent record, a 4 B reward, two 1 B flags and a 147 B observation staged
// in SMEM and written by one cp.async.bulk per 128-env tile.  Also times
// cudaMemcpy device->device of the same total bytes.  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sol_mix tools/sol_mix.cu && /tmp/sol_mix
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int TILE = 128, OBS = 147;

__global__ void __launch_bounds__(TILE) sol_step(const uint64_t* __restrict__ grid, uint64_t* __restrict__ agent,
                                                 const uint8_t* __restrict__ act, uint8_t* __restrict__ obs,
                                                 float* __restrict__ rew, uint8_t* __restrict__ term,
                                                 uint8_t* __restrict__ trunc) {
  __shared__ __align__(128) uint8_t s_obs[TILE * OBS];
  const int tid = threadIdx.x;
  const int64_t tile0 = (int64_t)blockIdx.x * TILE, e = tile0 + tid;
  uint64_t acc = agent[e] ^ act[e];
  const uint64_t* g = grid + tile0 * 8 + tid;
#pragma unroll
  for (int y = 0; y < 8; ++y) acc ^= g[y * TILE];
  // 36 words per env into the staging buffer (content irrelevant: the probe
  // measures traffic), written with the product's odd word stride
  uint32_t* s32 = reinterpret_cast<uint32_t*>(s_obs) + ((tid * OBS) >> 2);
#pragma unroll
  for (int i = 0; i < 36; ++i) s32[i] = (uint32_t)(acc >> (i & 31));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(obs + tile0 * OBS),
                 "r"((uint32_t)__cvta_generic_to_shared(s_obs)), "r"((uint32_t)(TILE * OBS))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  agent[e] = acc + 1;
  rew[e] = (float)(acc & 1);
  term[e] = (uint8_t)acc;
  trunc[e] = (uint8_t)(acc >> 8);
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

int main() {
  const int64_t n = 1 << 20, tiles = n / TILE;
  uint64_t *grid, *agent;
  uint8_t *act, *obs, *term, *trunc, *cpy_a, *cpy_b;
  float* rew;
  cudaMalloc(&grid, n * 64);
  cudaMalloc(&agent, n * 8);
  cudaMalloc(&act, n);
  cudaMalloc(&obs, n * OBS);
  cudaMalloc(&rew, n * 4);
  cudaMalloc(&term, n);
  cudaMalloc(&trunc, n);
  cudaMemset(grid, 1, n * 64);
  cudaMemset(agent, 0, n * 8);
  cudaMemset(act, 2, n);
  const int64_t bytes = n * (64 + 8 + 1 + 8 + 4 + 2 + OBS);  // 234 B per env-step
  cudaMalloc(&cpy_a, bytes / 2);
  cudaMalloc(&cpy_b, bytes / 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int K = 200;
  for (int i = 0; i < 20; ++i) sol_step<<<tiles, TILE>>>(grid, agent, act, obs, rew, term, trunc);
  cudaEventRecord(e0);
  for (int i = 0; i < K; ++i) sol_step<<<tiles, TILE>>>(grid, agent, act, obs, rew, term, trunc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_step;
  cudaEventElapsedTime(&ms_step, e0, e1);
  // plain copy of the same number of bytes (half read, half written)
  for (int i = 0; i < 5; ++i) cudaMemcpyAsync(cpy_b, cpy_a, bytes / 2, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e0);
  for (int i = 0; i < K; ++i) cudaMemcpyAsync(cpy_b, cpy_a, bytes / 2, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms_copy;
  cudaEventElapsedTime(&ms_copy, e0, e1);
  const double t_step = ms_step / 1e3 / K, t_copy = ms_copy / 1e3 / K;
  printf("{\"sol_step_us\": %.3f, \"sol_step_env_steps_per_s\": %.4g, \"sol_step_GBps\": %.1f, "
         "\"copy_us\": %.3f, \"copy_GBps\": %.1f, \"bytes_per_env_step\": 234, \"envs\": %lld, \"err\": \"%s\"}\n",
         t_step * 1e6, n / t_step, bytes / t_step / 1e9, t_copy * 1e6, bytes / t_copy / 1e9, (long long)n,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
