// capi.cu — host side of libnavix.so: the C ABI declared in include/navix.h.
//
// Argument validation, env-id parsing (Table 9 P:908-977 ids, Code 1 P:254
// grammar), state allocation, kernel launches on the caller's stream, and the
// canonical state export/import used for parity and checkpointing.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/navix.h"
#include "layout.h"

namespace navix {
cudaError_t launch_env_kernel(const EnvConfig& c, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s);
cudaError_t launch_sample_actions(uint8_t* out, int64_t n, int64_t steps, uint32_t env_begin, uint32_t t0,
                                  uint64_t seed, uint32_t n_actions, cudaStream_t s);
cudaError_t launch_stats_reduce(const unsigned long long* slots, long long* out8, cudaStream_t s);
cudaError_t launch_mission(const uint64_t* grid, const uint64_t* agent, int64_t n, int rw, int h, uint8_t* out,
                           cudaStream_t s);
}  // namespace navix

using namespace navix;

// Steps (rollouts) of at most this many envs run the small-batch kernels
// (navix_step_wide / navix_rollout_wide).  NAVIX_WIDE_MAX /
// NAVIX_WIDE_MAX_ROLLOUT override the defaults (A/B measurements).
static int64_t env_or(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  return e ? (int64_t)atoll(e) : dflt;
}
static int64_t default_wide_max() {
  static const int64_t v = env_or("NAVIX_WIDE_MAX", NAVIX_DEFAULT_WIDE_MAX);
  return v;
}
static int64_t default_wide_max_rollout() {
  static const int64_t v = env_or("NAVIX_WIDE_MAX_ROLLOUT", NAVIX_DEFAULT_WIDE_MAX_ROLLOUT);
  return v;
}

struct navix_env {
  EnvConfig cfg;
  navix_spec spec;
  StateLayout layout;
  int64_t n_total, env_begin, n;
  uint64_t seed;
  int device;
  int reward_mode;
  int obs_kind = 0;  // ObsKind (navix_set_observation)
  bool initialized = false;  // a reset or an import has written the state
  uint32_t reward_events = 7, termination_events = 7;  // navix_set_event_functions (R#42)
  float time_cost = 0.f, action_cost = 0.f;
  int64_t wide_max = default_wide_max();  // navix_set_small_batch_threshold
  int64_t wide_max_rollout = default_wide_max_rollout();
  uint8_t* state;
  bool owns_state;
  // navix_step_host staging (lazily allocated)
  uint8_t* h_actions = nullptr;
  uint8_t* h_obs = nullptr;
  float* h_reward = nullptr;
  uint8_t* h_term = nullptr;
  uint8_t* h_trunc = nullptr;
};

namespace {

thread_local std::string g_last_error;

navix_status fail(navix_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

navix_status cuda_fail(cudaError_t e, const char* what) {
  return fail(e == cudaErrorMemoryAllocation ? NAVIX_E_NOMEM : NAVIX_E_CUDA, "%s: %s (%s)", what,
              cudaGetErrorName(e), cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) changed = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

// Parse "<Family>-<params>" after stripping "Navix-"/"MiniGrid-" and "-v0".
// Returns 0 ok, 1 unknown, 2 known Table 9 id without a kernel in this build.
int parse_id(const char* env_id, EnvConfig* c) {
  if (!env_id) return 1;
  std::string id(env_id);
  for (const char* pre : {"Navix-", "MiniGrid-"})
    if (id.rfind(pre, 0) == 0) { id = id.substr(strlen(pre)); break; }
  if (id.size() > 3 && id.compare(id.size() - 3, 3, "-v0") == 0) id.resize(id.size() - 3);
  *c = EnvConfig{};
  int a = 0, b = 0;
  char tail = 0;
  auto sq = [&](const char* fmt) { return sscanf(id.c_str(), fmt, &a, &b, &tail) == 2 && a == b; };
  if (sq("Empty-Random-%dx%d%c")) {
    if (a != 5 && a != 6 && a != 8 && a != 16) return 1;
    *c = EnvConfig{FAM_EMPTY_RANDOM, a, a, 4 * a * a, 7, 0, 0, 0};
  } else if (id == "DistShift1" || id == "DistShift2") {  // [MG] DistShiftEnv 9x7 (R#33)
    *c = EnvConfig{id == "DistShift1" ? FAM_DISTSHIFT1 : FAM_DISTSHIFT2, 7, 9, 4 * 9 * 7, 7, 0, 0, 0};
  } else if (sscanf(id.c_str(), "SimpleCrossingS%dN%d%c", &a, &b, &tail) == 2 ||
             sscanf(id.c_str(), "Crossings-S%dN%d%c", &a, &b, &tail) == 2 ||
             sscanf(id.c_str(), "LavaCrossingS%dN%d%c", &a, &b, &tail) == 2) {
    // [MG] CrossingEnv (R#35): Table 8's SimpleCrossing = wall rivers;
    // Table 9's Crossings (R_2) = [MG]'s LavaCrossing, lava rivers
    if (!((a == 9 && b >= 1 && b <= 3) || (a == 11 && b == 5))) return 1;
    const int lava = id.rfind("SimpleCrossingS", 0) == 0 ? 0 : CROSSING_LAVA;
    *c = EnvConfig{FAM_CROSSING, a, a, 4 * a * a, 7, 0, 0, 0, b | lava};
  } else if (id == "FourRooms") {  // [MG] FourRoomsEnv at Table 9's 17x17, max_steps 100 (R#38)
    *c = EnvConfig{FAM_FOURROOMS, 17, 17, 100, 7, 0, 0, 0};
  } else if (sq("GoToDoor-%dx%d%c")) {  // [MG] GoToDoorEnv (R#37)
    if (a != 5 && a != 6 && a != 8) return 1;
    *c = EnvConfig{FAM_GOTODOOR, a, a, 4 * a * a, 7, 0, 0, 0};
  } else if (sq("Empty-%dx%d%c")) {
    if (a != 5 && a != 6 && a != 8 && a != 16) return 1;
    *c = EnvConfig{FAM_EMPTY, a, a, 4 * a * a, 7, 0, 0, 0};
  } else if (sq("DoorKey-%dx%d%c") || sq("DoorKey-Random-%dx%d%c")) {  // R#36
    if (a != 5 && a != 6 && a != 8 && a != 16) return 1;
    *c = EnvConfig{FAM_DOORKEY, a, a, 10 * a * a, 7, 0, 0, 0};
  } else if (sq("Dynamic-Obstacles-%dx%d%c") || sq("Dynamic-Obstacles-Random-%dx%d%c")) {
    if (a != 5 && a != 6 && a != 8 && a != 16) return 1;
    const int nob = a == 5 ? 2 : a == 6 ? 3 : a == 8 ? 4 : 8;  // R#6
    const int random_start = id.find("-Random-") != std::string::npos;  // R#40
    *c = EnvConfig{FAM_DYNOBS, a, a, 4 * a * a, 3, nob, 0, 0, random_start};
  } else if (sscanf(id.c_str(), "LavaGapS%d%c", &a, &tail) == 1 ||
             sscanf(id.c_str(), "LavaGap-S%d%c", &a, &tail) == 1) {  // Table 8 / Table 9 spellings
    if (a < 5 || a > 7) return 1;
    *c = EnvConfig{FAM_LAVAGAP, a, a, 4 * a * a, 7, 0, 0, 0};
  } else if (sscanf(id.c_str(), "KeyCorridorS%dR%d%c", &a, &b, &tail) == 2) {
    // the registered configurations (Table 9): S3R1-S3R3, S4R3, S5R3, S6R3
    if (!((a == 3 && b >= 1 && b <= 3) || (a >= 4 && a <= 6 && b == 3))) return 1;
    *c = EnvConfig{FAM_KEYCORRIDOR, (a - 1) * b + 1, (a - 1) * 3 + 1, 30 * a * a, 7, 0, a, b};
  } else {
    return 1;
  }
  return (c->height <= 24 && c->width <= 24) ? 0 : 2;
}

void fill_spec(const EnvConfig& c, navix_spec* s) {
  s->height = c.height;
  s->width = c.width;
  s->view = 7;
  s->n_actions = c.n_actions;
  s->max_steps = c.max_steps;
  s->obs_bytes = OBS_BYTES;
  // public NAVIX_FAMILY_* ids: DistShift1/2 share one, SimpleCrossing is 7
  s->family = c.family == FAM_DISTSHIFT2 ? FAM_DISTSHIFT1 : c.family == FAM_CROSSING ? 7 : c.family == FAM_GOTODOOR ? 8
              : c.family == FAM_FOURROOMS ? 9 : c.family;
  s->n_obstacles = c.n_obstacles;
  s->export_bytes = 3 * c.height * c.width + 12 + 2 * c.n_obstacles + (c.family == FAM_GOTODOOR ? 2 : 0);
}

KernelArgs make_args(navix_env* h) {
  KernelArgs a{};
  uint8_t* s = h->state;
  a.grid = reinterpret_cast<uint64_t*>(s + h->layout.grid_off);
  a.agent = reinterpret_cast<uint64_t*>(s + h->layout.agent_off);
  a.episode = reinterpret_cast<uint32_t*>(s + h->layout.episode_off);
  a.balls = reinterpret_cast<uint64_t*>(s + h->layout.balls_off);
  a.stats = reinterpret_cast<unsigned long long*>(s + h->layout.stats_off);
  a.sched = reinterpret_cast<unsigned int*>(s + h->layout.sched_off);
  a.n = h->n;
  a.env_begin = (uint32_t)h->env_begin;
  a.key_lo = (uint32_t)h->seed;
  a.key_hi = (uint32_t)(h->seed >> 32);
  a.reward_mode = h->reward_mode;
  a.time_cost = h->time_cost;
  a.action_cost = h->action_cost;
  a.gen_param = h->cfg.gen_param;
  a.obs_kind = h->obs_kind;
  a.reward_events = h->reward_events;
  a.termination_events = h->termination_events;
  a.wide_max = h->wide_max;
  a.wide_max_rollout = h->wide_max_rollout;
  return a;
}

navix_status launch(navix_env* h, int mode, KernelArgs& a, void* stream) {
  a.bulk_obs = (reinterpret_cast<uintptr_t>(a.obs) & 15u) == 0;
  a.bulk_act = (reinterpret_cast<uintptr_t>(a.actions) & 15u) == 0;
  DeviceGuard dg(h->device);
  cudaError_t e = launch_env_kernel(h->cfg, mode, a, h->layout.n_tiles, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "navix kernel launch");
  return NAVIX_OK;
}

// canonical (type, colour, state) -> internal cell byte (layout.h); false if illegal
bool to_cell(const uint8_t* t, uint8_t* out) {
  const uint8_t type = t[0], col = t[1], st = t[2];
  if (col > 5 || st > 2) return false;
  if (type != 4 && st != 0) return false;
  switch (type) {
    case 1: if (col) return false; *out = CELL_EMPTY; return true;
    case 2: *out = make_cell(K_WALL, col); return true;
    case 3: *out = make_cell(K_FLOOR, col); return true;
    case 4: *out = make_cell(st == 0 ? K_DOOR_OPEN : st == 1 ? K_DOOR_CLOSED : K_DOOR_LOCKED, col); return true;
    case 5: *out = make_cell(K_KEY, col); return true;
    case 6: *out = make_cell(K_BALL, col); return true;
    case 7: *out = make_cell(K_BOX, col); return true;
    case 8: *out = make_cell(K_GOAL, col); return true;
    case 9: *out = make_cell(K_LAVA, col); return true;
    default: return false;
  }
}

void from_cell(uint8_t c, uint8_t* t) {
  const uint8_t kind = c & 15;
  t[0] = kind >= 11 ? 4 : kind;
  t[1] = (c >> 4) & 7;
  t[2] = kind >= 11 ? kind - 10 : 0;
}

bool walkable_kind(uint8_t kind) { return (0x31Au >> kind) & 1u; }

// levelgen.cuh STATIC_LAYOUT / template_plane, for the run-time config of a handle
bool static_layout_family(int f) {
  return f == FAM_DYNOBS || f == FAM_EMPTY || f == FAM_EMPTY_RANDOM || f == FAM_DISTSHIFT1 || f == FAM_DISTSHIFT2;
}
uint8_t template_cell(const EnvConfig& c, int x, int y) {
  const int W = c.width, H = c.height;
  if (x == 0 || y == 0 || x == W - 1 || y == H - 1) return CELL_WALL;
  if (c.family == FAM_DISTSHIFT1 || c.family == FAM_DISTSHIFT2) {  // R#33
    const int strip2 = c.family == FAM_DISTSHIFT1 ? 2 : 5;
    if (x == W - 2 && y == 1) return CELL_GOAL;
    if (x >= 3 && x < W - 3 && (y == 1 || y == strip2)) return CELL_LAVA;
    return CELL_EMPTY;
  }
  return (x == W - 2 && y == H - 2) ? CELL_GOAL : CELL_EMPTY;
}

}  // namespace

extern "C" {

const char* navix_last_error(void) { return g_last_error.c_str(); }

#ifndef NAVIX_BUILD_ID
#define NAVIX_BUILD_ID "unknown0unknown0"
#endif
// the marker string lets build.py read the id from the .so without loading it
__attribute__((used)) static const char k_build_id[] = "NAVIX_BUILD_ID=" NAVIX_BUILD_ID;
const char* navix_build_id(void) { return k_build_id + 15; }

navix_status navix_spec_of(const char* env_id, navix_spec* out) {
  if (!out) return fail(NAVIX_E_INVALID_ARG, "navix_spec_of: null out");
  EnvConfig c;
  const int r = parse_id(env_id, &c);
  if (r == 1) return fail(NAVIX_E_UNKNOWN_ENV, "unknown env id '%s' (Table 9 ids, e.g. Navix-DoorKey-8x8-v0)",
                          env_id ? env_id : "(null)");
  fill_spec(c, out);
  if (r == 2) return fail(NAVIX_E_UNSUPPORTED, "env id '%s' has a %dx%d grid; this build supports <= 24x24",
                          env_id, c.height, c.width);
  return NAVIX_OK;
}

size_t navix_state_bytes(const char* env_id, int64_t num_envs) {
  EnvConfig c;
  if (num_envs <= 0 || parse_id(env_id, &c) != 0) return 0;
  return make_layout(c, num_envs).total;
}

navix_status navix_create_shard(const char* env_id, int64_t num_envs_total, int64_t env_begin,
                                int64_t num_envs_local, uint64_t seed, int device, void* state_dev,
                                int reward_mode, navix_env** out) {
  if (!out) return fail(NAVIX_E_INVALID_ARG, "navix_create_shard: null out");
  *out = nullptr;
  EnvConfig c;
  const int r = parse_id(env_id, &c);
  if (r == 1) return fail(NAVIX_E_UNKNOWN_ENV, "unknown env id '%s'", env_id ? env_id : "(null)");
  if (r == 2) return fail(NAVIX_E_UNSUPPORTED, "env id '%s' (%dx%d) has no kernel in this build", env_id,
                          c.height, c.width);
  if (num_envs_local <= 0 || num_envs_total <= 0)
    return fail(NAVIX_E_INVALID_ARG, "num_envs must be positive (got local %lld, total %lld)",
                (long long)num_envs_local, (long long)num_envs_total);
  if (env_begin < 0 || env_begin + num_envs_local > num_envs_total)
    return fail(NAVIX_E_INVALID_ARG, "shard [%lld, %lld) outside [0, %lld)", (long long)env_begin,
                (long long)(env_begin + num_envs_local), (long long)num_envs_total);
  if (num_envs_total > (int64_t)UINT32_MAX) return fail(NAVIX_E_INVALID_ARG, "num_envs_total exceeds 2^32");
  if (reward_mode != NAVIX_REWARD_MINIGRID && reward_mode != NAVIX_REWARD_NAVIX)
    return fail(NAVIX_E_INVALID_ARG, "reward_mode must be 0 (minigrid) or 1 (navix)");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(NAVIX_E_INVALID_ARG, "device %d not in [0, %d)", device, ndev);
  if (state_dev && (reinterpret_cast<uintptr_t>(state_dev) & 255u))
    return fail(NAVIX_E_INVALID_ARG, "state buffer must be 256-byte aligned");
  navix_env* h = new navix_env();
  h->cfg = c;
  fill_spec(c, &h->spec);
  h->layout = make_layout(c, num_envs_local);
  h->n_total = num_envs_total;
  h->env_begin = env_begin;
  h->n = num_envs_local;
  h->seed = seed;
  h->device = device;
  h->reward_mode = reward_mode;
  if (state_dev) {
    h->state = static_cast<uint8_t*>(state_dev);
    h->owns_state = false;
  } else {
    DeviceGuard dg(device);
    e = cudaMalloc(&h->state, h->layout.total);
    if (e != cudaSuccess) {
      delete h;
      return cuda_fail(e, "cudaMalloc(state)");
    }
    h->owns_state = true;
  }
  {  // scheduler and statistics start at zero even before the first reset
    DeviceGuard dg(device);
    e = cudaMemset(h->state + h->layout.stats_off, 0, h->layout.total - h->layout.stats_off);
    if (e == cudaSuccess && (static_layout_family(h->cfg.family) || h->cfg.family == FAM_LAVAGAP ||
                             h->cfg.family == FAM_CROSSING || (h->cfg.family == FAM_DOORKEY && h->cfg.width <= 8))) {
      // the per-device visibility table of the static-layout families
      // (step_kernel.cuh obs_table_kernel); idempotent, outside any capture
      KernelArgs a{};
      a.obs_kind = OBS_SYMBOLIC;
      e = launch_env_kernel(h->cfg, MODE_OBS_TABLE, a, 1, nullptr);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) {
      if (h->owns_state) cudaFree(h->state);
      delete h;
      return cuda_fail(e, "cudaMemset(stats) / observation table");
    }
  }
  *out = h;
  return NAVIX_OK;
}

navix_status navix_create(const char* env_id, int64_t num_envs, uint64_t seed, navix_env** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  return navix_create_shard(env_id, num_envs, 0, num_envs, seed, dev, nullptr, NAVIX_REWARD_MINIGRID, out);
}

navix_status navix_reset(navix_env* h, uint8_t* obs, void* stream) {
  if (!h || !obs) return fail(NAVIX_E_INVALID_ARG, "navix_reset: null handle or obs");
  {
    DeviceGuard dg(h->device);
    cudaError_t e = cudaMemsetAsync(h->state + h->layout.stats_off, 0, h->layout.total - h->layout.stats_off,
                                    (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(stats)");
  }
  KernelArgs a = make_args(h);
  a.obs = obs;
  const navix_status st = launch(h, MODE_RESET, a, stream);
  if (st == NAVIX_OK) h->initialized = true;
  return st;
}

navix_status navix_reset_seed(navix_env* h, uint64_t seed, uint8_t* obs, void* stream) {
  if (!h || !obs) return fail(NAVIX_E_INVALID_ARG, "navix_reset_seed: null handle or obs");
  h->seed = seed;  // the Philox key of every later level / obstacle draw
  return navix_reset(h, obs, stream);
}

navix_status navix_step(navix_env* h, const uint8_t* actions, uint8_t* obs, float* reward, uint8_t* terminated,
                        uint8_t* truncated, void* stream) {
  if (!h || !actions || !obs || !reward || !terminated || !truncated)
    return fail(NAVIX_E_INVALID_ARG, "navix_step: null argument");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_step: call navix_reset (or navix_state_import) first");
  KernelArgs a = make_args(h);
  a.actions = actions;
  a.obs = obs;
  a.reward = reward;
  a.terminated = terminated;
  a.truncated = truncated;
  return launch(h, MODE_STEP, a, stream);
}

navix_status navix_rollout(navix_env* h, const uint8_t* actions, int64_t steps, uint8_t* obs, float* reward,
                           uint8_t* terminated, uint8_t* truncated, void* stream) {
  if (!h || !actions || !obs || !reward || !terminated || !truncated)
    return fail(NAVIX_E_INVALID_ARG, "navix_rollout: null argument");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_rollout: call navix_reset (or navix_state_import) first");
  if (steps <= 0) return fail(NAVIX_E_INVALID_ARG, "navix_rollout: steps must be positive (got %lld)", (long long)steps);
  KernelArgs a = make_args(h);
  a.actions = actions;
  a.obs = obs;
  a.reward = reward;
  a.terminated = terminated;
  a.truncated = truncated;
  a.rollout_steps = steps;
  return launch(h, MODE_ROLLOUT, a, stream);
}

navix_status navix_rollout_random(navix_env* h, uint64_t action_seed, int64_t t0, int64_t steps, uint8_t* obs,
                                  float* reward, uint8_t* terminated, uint8_t* truncated, void* stream) {
  if (!h || !obs || !reward || !terminated || !truncated)
    return fail(NAVIX_E_INVALID_ARG, "navix_rollout_random: null argument");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_rollout_random: call navix_reset (or navix_state_import) first");
  if (steps <= 0 || t0 < 0)
    return fail(NAVIX_E_INVALID_ARG, "navix_rollout_random: steps must be positive and t0 >= 0");
  KernelArgs a = make_args(h);
  a.actions = nullptr;  // in-kernel policy
  a.act_key_lo = (uint32_t)action_seed;
  a.act_key_hi = (uint32_t)(action_seed >> 32);
  a.act_t0 = (uint32_t)t0;
  a.obs = obs;
  a.reward = reward;
  a.terminated = terminated;
  a.truncated = truncated;
  a.rollout_steps = steps;
  return launch(h, MODE_ROLLOUT, a, stream);
}

navix_status navix_set_reward_costs(navix_env* h, float time_cost, float action_cost) {
  if (!h) return fail(NAVIX_E_INVALID_ARG, "navix_set_reward_costs: null handle");
  if (!(time_cost >= 0.f && time_cost < 1e30f) || !(action_cost >= 0.f && action_cost < 1e30f))
    return fail(NAVIX_E_INVALID_ARG, "reward costs must be finite and >= 0");
  h->time_cost = time_cost;
  h->action_cost = action_cost;
  return NAVIX_OK;
}

navix_status navix_set_event_functions(navix_env* h, uint32_t reward_events, uint32_t termination_events) {
  if (!h) return fail(NAVIX_E_INVALID_ARG, "navix_set_event_functions: null handle");
  if ((reward_events | termination_events) & ~7u)
    return fail(NAVIX_E_INVALID_ARG, "event masks use bits 0-2 only (got %#x, %#x)", reward_events, termination_events);
  h->reward_events = reward_events;
  h->termination_events = termination_events;
  return NAVIX_OK;
}

navix_status navix_set_small_batch_threshold(navix_env* h, int64_t max_envs) {
  if (!h) return fail(NAVIX_E_INVALID_ARG, "navix_set_small_batch_threshold: null handle");
  if (max_envs < 0) return fail(NAVIX_E_INVALID_ARG, "threshold must be >= 0 (0 disables the small-batch kernel)");
  h->wide_max = max_envs;
  h->wide_max_rollout = max_envs;
  return NAVIX_OK;
}

navix_status navix_set_observation(navix_env* h, int kind) {
  if (!h) return fail(NAVIX_E_INVALID_ARG, "navix_set_observation: null handle");
  if (kind != NAVIX_OBS_SYMBOLIC && kind != NAVIX_OBS_CATEGORICAL)
    return fail(NAVIX_E_INVALID_ARG, "unknown observation kind %d", kind);
  h->obs_kind = kind;
  return NAVIX_OK;
}

navix_status navix_observe_full(navix_env* h, uint8_t* out, void* stream) {
  if (!h || !out) return fail(NAVIX_E_INVALID_ARG, "navix_observe_full: null argument");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_observe_full: call navix_reset (or navix_state_import) first");
  KernelArgs a = make_args(h);
  a.obs = out;
  return launch(h, MODE_FULL_OBS, a, stream);
}

navix_status navix_observe(navix_env* h, uint8_t* obs, void* stream) {
  if (!h || !obs) return fail(NAVIX_E_INVALID_ARG, "navix_observe: null argument");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_observe: call navix_reset (or navix_state_import) first");
  KernelArgs a = make_args(h);
  a.obs = obs;
  return launch(h, MODE_OBSERVE, a, stream);
}

navix_status navix_sample_actions(navix_env* h, uint64_t action_seed, int64_t t0, int64_t steps, uint8_t* out,
                                  void* stream) {
  if (!h || !out || steps <= 0 || t0 < 0) return fail(NAVIX_E_INVALID_ARG, "navix_sample_actions: bad argument");
  DeviceGuard dg(h->device);
  cudaError_t e = launch_sample_actions(out, h->n, steps, (uint32_t)h->env_begin, (uint32_t)t0, action_seed,
                                        (uint32_t)h->cfg.n_actions, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sample_actions launch");
  return NAVIX_OK;
}

navix_status navix_step_host(navix_env* h, const uint8_t* actions, uint8_t* obs, float* reward,
                             uint8_t* terminated, uint8_t* truncated, void* stream) {
  if (!h || !actions || !obs || !reward || !terminated || !truncated)
    return fail(NAVIX_E_INVALID_ARG, "navix_step_host: null argument");
  DeviceGuard dg(h->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t n = (size_t)h->n;
  cudaError_t e;
  if (!h->h_actions) {
    // one allocation: actions | obs (16-B aligned) | reward | terminated | truncated
    uint8_t* base = nullptr;
    const size_t obs_off = align_up(n, 256), rew_off = align_up(obs_off + n * OBS_BYTES, 256);
    const size_t term_off = align_up(rew_off + 4 * n, 256), trunc_off = align_up(term_off + n, 256);
    e = cudaMalloc(&base, trunc_off + n);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(step_host staging)");
    h->h_actions = base;
    h->h_obs = base + obs_off;
    h->h_reward = reinterpret_cast<float*>(base + rew_off);
    h->h_term = base + term_off;
    h->h_trunc = base + trunc_off;
  }
  if ((e = cudaMemcpyAsync(h->h_actions, actions, n, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "H2D actions");
  navix_status st = navix_step(h, h->h_actions, h->h_obs, h->h_reward, h->h_term, h->h_trunc, stream);
  if (st != NAVIX_OK) return st;
  if ((e = cudaMemcpyAsync(obs, h->h_obs, n * obs_record_bytes(h->obs_kind), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(reward, h->h_reward, n * 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(terminated, h->h_term, n, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(truncated, h->h_trunc, n, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "D2H step outputs");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return NAVIX_OK;
}

navix_status navix_observe_mission(navix_env* h, uint8_t* out, void* stream) {
  if (!h || !out) return fail(NAVIX_E_INVALID_ARG, "navix_observe_mission: null argument");
  if (h->cfg.family != FAM_GOTODOOR)
    return fail(NAVIX_E_INVALID_ARG, "navix_observe_mission: only GoToDoor has a mission");
  if (!h->initialized) return fail(NAVIX_E_INVALID_ARG, "navix_observe_mission: call navix_reset first");
  DeviceGuard dg(h->device);
  cudaError_t e = launch_mission(reinterpret_cast<const uint64_t*>(h->state + h->layout.grid_off),
                                 reinterpret_cast<const uint64_t*>(h->state + h->layout.agent_off), h->n,
                                 row_planes(h->cfg.width), h->cfg.height, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "mission launch");
  return NAVIX_OK;
}

navix_status navix_stats(navix_env* h, int64_t* out8, void* stream) {
  if (!h || !out8) return fail(NAVIX_E_INVALID_ARG, "navix_stats: null argument");
  DeviceGuard dg(h->device);
  cudaError_t e = launch_stats_reduce(reinterpret_cast<const unsigned long long*>(h->state + h->layout.stats_off),
                                      reinterpret_cast<long long*>(out8), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "stats launch");
  return NAVIX_OK;
}

navix_status navix_state_export(navix_env* h, void* host, size_t cap, size_t* written) {
  if (!h) return fail(NAVIX_E_INVALID_ARG, "navix_state_export: null handle");
  const EnvConfig& c = h->cfg;
  const size_t per = (size_t)h->spec.export_bytes, need = per * (size_t)h->n;
  if (written) *written = need;
  if (!host) return NAVIX_OK;  // size query
  if (cap < need) return fail(NAVIX_E_INVALID_ARG, "export buffer too small (%zu < %zu)", cap, need);
  DeviceGuard dg(h->device);
  const StateLayout& L = h->layout;
  const int RW = row_planes(c.width), HP = c.height * RW;
  std::vector<uint64_t> grid((size_t)L.n_pad * HP), agent((size_t)L.n_pad);
  std::vector<uint32_t> episode((size_t)L.n_pad);
  std::vector<uint64_t> balls(c.family == FAM_DYNOBS ? (size_t)L.n_pad : 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
  if ((e = cudaMemcpy(grid.data(), h->state + L.grid_off, grid.size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(agent.data(), h->state + L.agent_off, agent.size() * 8, cudaMemcpyDeviceToHost)) !=
          cudaSuccess ||
      (e = cudaMemcpy(episode.data(), h->state + L.episode_off, episode.size() * 4, cudaMemcpyDeviceToHost)) !=
          cudaSuccess)
    return cuda_fail(e, "export D2H");
  if (!balls.empty() &&
      (e = cudaMemcpy(balls.data(), h->state + L.balls_off, balls.size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cuda_fail(e, "export D2H balls");
  uint8_t* o = static_cast<uint8_t*>(host);
  for (int64_t i = 0; i < h->n; ++i) {
    const int64_t tile = i / TILE, lane = slot_of_env((int)(i % TILE)), si = tile * TILE + lane;
    uint8_t cells[24][24];
    for (int y = 0; y < c.height; ++y)
      for (int x = 0; x < c.width; ++x)
        cells[y][x] = (uint8_t)(grid[(size_t)(tile * HP + y * RW + x / 8) * TILE + lane] >> (8 * (x % 8)));
    if (c.family == FAM_DYNOBS)
      for (int b = 0; b < c.n_obstacles; ++b) {
        const uint32_t p = (uint32_t)(balls[si] >> (8 * b)) & 0xFF;
        if (p) cells[ball_y(c.width, p)][ball_x(c.width, p)] = make_cell(K_BALL, COL_BLUE);
      }
    uint8_t* p = o + (size_t)i * per;
    for (int y = 0; y < c.height; ++y)
      for (int x = 0; x < c.width; ++x, p += 3) from_cell(cells[y][x], p);
    const uint64_t r = agent[si];
    p[0] = (uint8_t)r;
    p[1] = (uint8_t)(r >> 8);
    p[2] = (uint8_t)(r >> 16);
    uint8_t ct[3];
    from_cell((uint8_t)(r >> 24), ct);
    p[3] = ct[0];
    p[4] = ct[1];
    p[5] = (uint8_t)(r >> 32);
    p[6] = (uint8_t)(r >> 40);
    memcpy(p + 7, &episode[si], 4);
    p[11] = (uint8_t)((r >> 48) & 1);
    p += 12;
    for (int b = 0; b < c.n_obstacles; ++b, p += 2) {
      const uint32_t q = (uint32_t)(balls[si] >> (8 * b)) & 0xFF;
      p[0] = (uint8_t)ball_x(c.width, q);
      p[1] = (uint8_t)ball_y(c.width, q);
    }
    if (c.family == FAM_GOTODOOR) {  // target door: agent record byte 7 = (x << 4) | y
      p[0] = (uint8_t)(r >> 60);
      p[1] = (uint8_t)((r >> 56) & 15);
    }
  }
  return NAVIX_OK;
}

navix_status navix_state_import(navix_env* h, const void* host, size_t n_bytes) {
  if (!h || !host) return fail(NAVIX_E_INVALID_ARG, "navix_state_import: null argument");
  const EnvConfig& c = h->cfg;
  const size_t per = (size_t)h->spec.export_bytes;
  if (n_bytes != per * (size_t)h->n)
    return fail(NAVIX_E_INVALID_ARG, "import size %zu != %lld envs x %zu bytes", n_bytes, (long long)h->n, per);
  const StateLayout& L = h->layout;
  const int H = c.height, W = c.width, RW = row_planes(W);
  std::vector<uint64_t> grid((size_t)L.n_pad * H * RW, 0), agent((size_t)L.n_pad, 0), balls((size_t)L.n_pad, 0);
  std::vector<uint32_t> episode((size_t)L.n_pad, 0);
  const uint8_t* in = static_cast<const uint8_t*>(host);
  for (int64_t i = 0; i < h->n; ++i) {
    const uint8_t* p = in + (size_t)i * per;
    uint8_t cells[24][24] = {};
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x, p += 3) {
        if (!to_cell(p, &cells[y][x]))
          return fail(NAVIX_E_INVALID_ARG, "env %lld: illegal cell code (%d,%d,%d) at (%d,%d)", (long long)i, p[0],
                      p[1], p[2], x, y);
        const bool border = x == 0 || y == 0 || x == W - 1 || y == H - 1;
        if (border && c.family != FAM_GOTODOOR && (cells[y][x] & 15) != K_WALL)
          return fail(NAVIX_E_INVALID_ARG, "env %lld: border cell (%d,%d) is not a wall (R#12)", (long long)i, x, y);
      }
    const int ax = p[0], ay = p[1], dir = p[2];
    const int m = c.family == FAM_GOTODOOR ? 0 : 1;  // GoToDoor: open grid edge (R#37)
    if (ax < m || ay < m || ax > W - 1 - m || ay > H - 1 - m || dir > 3)
      return fail(NAVIX_E_INVALID_ARG, "env %lld: agent (%d,%d,%d) not an interior pose", (long long)i, ax, ay, dir);
    if (!walkable_kind(cells[ay][ax] & 15))
      return fail(NAVIX_E_INVALID_ARG, "env %lld: agent stands on a non-walkable cell", (long long)i);
    uint8_t carry;
    const uint8_t ct[3] = {p[3], p[4], 0};
    if (!to_cell(ct, &carry) || !(carry == CELL_EMPTY || ((0xE0u >> (carry & 15)) & 1u)))
      return fail(NAVIX_E_INVALID_ARG, "env %lld: illegal carried object (%d,%d)", (long long)i, p[3], p[4]);
    const uint32_t sc = p[5] | (p[6] << 8);
    uint32_t ep;
    memcpy(&ep, p + 7, 4);
    const uint8_t pd = p[11];
    if (sc > (uint32_t)c.max_steps || pd > 1)
      return fail(NAVIX_E_INVALID_ARG, "env %lld: step_count %u / prev_done %u out of range", (long long)i, sc, pd);
    p += 12;
    uint64_t bl = 0;
    for (int b = 0; b < c.n_obstacles; ++b, p += 2) {
      const int bx = p[0], by = p[1];
      if (bx < 1 || by < 1 || bx > W - 2 || by > H - 2 || cells[by][bx] != make_cell(K_BALL, COL_BLUE))
        return fail(NAVIX_E_INVALID_ARG, "env %lld: obstacle %d at (%d,%d) is not a blue ball", (long long)i, b, bx,
                    by);
      for (int q = 0; q < b; ++q)
        if (((bl >> (8 * q)) & 0xFF) == (uint64_t)ball_code(W, bx, by))
          return fail(NAVIX_E_INVALID_ARG, "env %lld: duplicate obstacle", (long long)i);
      bl |= (uint64_t)ball_code(W, bx, by) << (8 * b);
    }
    uint64_t target = 0;
    if (c.family == FAM_GOTODOOR) {
      if (p[0] >= W || p[1] >= H)
        return fail(NAVIX_E_INVALID_ARG, "env %lld: target (%d,%d) outside the grid", (long long)i, p[0], p[1]);
      target = (uint64_t)((p[0] << 4) | p[1]) << 56;
    }
    for (int b = 0; b < c.n_obstacles; ++b) {  // balls live outside the HBM grid
      const uint32_t q = (uint32_t)(bl >> (8 * b)) & 0xFF;
      cells[ball_y(W, q)][ball_x(W, q)] = CELL_EMPTY;
    }
    // static-layout families: agent-record flag bit 1 (layout.h) marks a
    // layout equal to the generator's template (levelgen.cuh template_plane),
    // which the step kernel then knows without reading it
    uint64_t tmpl_flag = 0;
    if (static_layout_family(c.family)) {
      bool same = true;
      for (int y = 0; y < H && same; ++y)
        for (int x = 0; x < W && same; ++x) same = cells[y][x] == template_cell(c, x, y);
      tmpl_flag = same ? 2 : 0;
    }
    // DoorKey: a generated layout's opaque cells (levelgen.cuh
    // LAYOUT_KEYED_VIS) — flag bit 2 and byte 7 = (split << 4) | door_y
    uint64_t layout_key = 0;
    if (c.family == FAM_DOORKEY && W <= 8) {
      int split = -1, door_y = -1, doors = 0;
      bool ok = true;
      for (int y = 1; y < H - 1 && ok; ++y)
        for (int x = 1; x < W - 1 && ok; ++x) {
          const int k = cells[y][x] & 15;
          const bool door = k == K_DOOR_OPEN || k == K_DOOR_CLOSED || k == K_DOOR_LOCKED;
          if (k != K_WALL && !door) continue;
          if (split < 0) split = x;
          ok = x == split;
          if (door) { ++doors; door_y = y; }
        }
      if (ok && split >= 2 && split <= W - 3 && doors == 1 && door_y >= 1 && door_y <= W - 3) {
        for (int y = 1; y < H - 1 && ok; ++y) {
          const int k = cells[y][split] & 15;
          ok = y == door_y || k == K_WALL;
        }
        if (ok) layout_key = (4ull << 48) | ((uint64_t)((split << 4) | door_y) << 56);
      }
    }
    // LavaGap / Crossings (levelgen.cuh BORDER_OPACITY): no door and no opaque
    // cell inside the border — flag bit 2, key 0
    if (c.family == FAM_LAVAGAP || c.family == FAM_CROSSING) {
      bool ok = true;
      for (int y = 1; y < H - 1 && ok; ++y)
        for (int x = 1; x < W - 1 && ok; ++x) {
          const int k = cells[y][x] & 15;
          ok = k != K_WALL && k != K_DOOR_OPEN && k != K_DOOR_CLOSED && k != K_DOOR_LOCKED;
        }
      if (ok) layout_key = 4ull << 48;
    }
    const int64_t tile = i / TILE, lane = slot_of_env((int)(i % TILE)), si = tile * TILE + lane;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        grid[(size_t)(tile * H * RW + y * RW + x / 8) * TILE + lane] |= (uint64_t)cells[y][x] << (8 * (x % 8));
    agent[si] = (uint64_t)ax | ((uint64_t)ay << 8) | ((uint64_t)dir << 16) | ((uint64_t)carry << 24) |
               ((uint64_t)sc << 32) | ((uint64_t)(pd | tmpl_flag) << 48) | target | layout_key;
    episode[si] = ep;
    balls[si] = bl;
  }
  DeviceGuard dg(h->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
  if ((e = cudaMemcpy(h->state + L.grid_off, grid.data(), grid.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(h->state + L.agent_off, agent.data(), agent.size() * 8, cudaMemcpyHostToDevice)) !=
          cudaSuccess ||
      (e = cudaMemcpy(h->state + L.episode_off, episode.data(), episode.size() * 4, cudaMemcpyHostToDevice)) !=
          cudaSuccess)
    return cuda_fail(e, "import H2D");
  if (c.family == FAM_DYNOBS &&
      (e = cudaMemcpy(h->state + L.balls_off, balls.data(), balls.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "import H2D balls");
  // pageable host -> device cudaMemcpy may return before the DMA lands, and
  // the legacy stream does not order against non-blocking streams: finish here
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_fail(e, "cudaDeviceSynchronize");
  h->initialized = true;
  return NAVIX_OK;
}

navix_status navix_info(navix_env* h, int64_t* out4) {
  if (!h || !out4) return fail(NAVIX_E_INVALID_ARG, "navix_info: null argument");
  out4[0] = h->n;
  out4[1] = h->env_begin;
  out4[2] = h->n_total;
  out4[3] = h->device;
  return NAVIX_OK;
}

void navix_destroy(navix_env* h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  if (h->owns_state && h->state) cudaFree(h->state);
  if (h->h_actions) cudaFree(h->h_actions);
  delete h;
}

}  // extern "C"
