// tools/launch_floor.cu — the small-batch floor of a graph-replayed step:
// per-launch time of (a) an empty kernel, (b) an empty kernel launched with
// programmatic dependent launch (PDL, as the step kernels are), (c) a kernel
// moving exactly one DoorKey-8x8 step's bytes (64 B grid + 8 B agent + 1 B
// action in; 8 B agent + 147 B obs via one TMA bulk store per tile + 4 B
// reward + 2 B flags out) with PDL, (d) (c) plus a dependent ALU chain of
// CHAIN instructions per thread.  Grid = ceil(N / 128) CTAs of 128 threads.
// Prints one JSON line per N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_floor tools/launch_floor.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int TILE = 128, OBS = 147;

__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 1000) *p = 1;
}
__global__ void empty_pdl(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p && threadIdx.x == 1000) *p = 1;
}

template <int CHAIN>
__global__ void __launch_bounds__(TILE) bytes_pdl(const uint64_t* __restrict__ grid, uint64_t* __restrict__ agent,
                                                  const uint8_t* __restrict__ act, uint8_t* __restrict__ obs,
                                                  float* __restrict__ rew, uint8_t* __restrict__ term, int64_t n) {
  __shared__ __align__(128) uint8_t s_obs[TILE * OBS];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int tid = threadIdx.x;
  const int64_t tile0 = (int64_t)blockIdx.x * TILE, e = tile0 + tid;
  uint64_t acc = agent[e] ^ act[e];
  const uint64_t* g = grid + tile0 * 8 + tid;
#pragma unroll
  for (int y = 0; y < 8; ++y) acc ^= g[y * TILE];
  uint32_t x = (uint32_t)acc, y = (uint32_t)(acc >> 32);
#pragma unroll 1
  for (int i = 0; i < CHAIN / 4; ++i) {  // 4 dependent ALU ops per iteration (+ loop overhead)
    x = __byte_perm(x, y, 0x5140);
    y = x ^ (y >> 3);
    x = (x + y) | 1u;
    y = __funnelshift_l(x, y, 5);
  }
  acc ^= ((uint64_t)y << 32) | x;
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
  agent[e] = acc;
  rew[e] = (float)(acc & 0xFF);
  term[e] = (uint8_t)acc;
  term[n + e] = (uint8_t)(acc >> 8);
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

template <class F>
static float time_graph(F launch_one, int iters, cudaStream_t s) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < iters; ++i) launch_one();
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best * 1000.f / iters;  // us per launch
}

template <class K, class... Args>
static void launch_pdl(K kernel, unsigned grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TILE);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

int main() {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int64_t NMAX = 1 << 16;
  uint64_t *grid, *agent;
  uint8_t *act, *obs, *term;
  float* rew;
  cudaMalloc(&grid, NMAX * 64);
  cudaMalloc(&agent, NMAX * 8);
  cudaMalloc(&act, NMAX);
  cudaMalloc(&obs, NMAX * OBS);
  cudaMalloc(&rew, NMAX * 4);
  cudaMalloc(&term, NMAX * 2);
  cudaMemset(grid, 0, NMAX * 64);
  cudaMemset(agent, 0, NMAX * 8);
  cudaMemset(act, 0, NMAX);
  const int iters = 1000;
  for (int64_t n : {128LL, 2048LL, 16384LL, 65536LL}) {
    const unsigned g = (unsigned)((n + TILE - 1) / TILE);
    const float t_empty = time_graph([&] { empty_kernel<<<g, TILE, 0, s>>>(nullptr); }, iters, s);
    const float t_pdl = time_graph([&] { launch_pdl(empty_pdl, g, s, (int*)nullptr); }, iters, s);
    const float t_bytes = time_graph([&] { launch_pdl(bytes_pdl<0>, g, s, grid, agent, act, obs, rew, term, n); },
                                     iters, s);
    const float t_c256 = time_graph([&] { launch_pdl(bytes_pdl<256>, g, s, grid, agent, act, obs, rew, term, n); },
                                    iters, s);
    const float t_c1024 = time_graph([&] { launch_pdl(bytes_pdl<1024>, g, s, grid, agent, act, obs, rew, term, n); },
                                     iters, s);
    printf("{\"n\": %lld, \"us_empty\": %.3f, \"us_empty_pdl\": %.3f, \"us_bytes_pdl\": %.3f, "
           "\"us_bytes_chain256_pdl\": %.3f, \"us_bytes_chain1024_pdl\": %.3f, \"err\": \"%s\"}\n",
           (long long)n, t_empty, t_pdl, t_bytes, t_c256, t_c1024, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
