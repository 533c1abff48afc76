/* navix.h — C ABI of libnavix.so: a B200-native batched MiniGrid step.
 *
 * The operation is one batched step of NAVIX (arXiv 2407.19396): for each of
 * n independent environments, `step(timestep, action)` with auto-reset
 * (§3.2.2, Code 1 P:264 "autoresets when done"), composed
 * of the systems of Table 3: intervention I, transition
 * mu (moving obstacles), observation O = symbolic_first_person
 * (Table 5; or categorical_first_person, R#41), reward R (Eq. (1), Table 6) and
 * termination gamma (Table 7; "all environments terminate when the
 * reward is not 0").  The environments are those of Table 9
 * with MiniGrid's rules.  Readings where the paper is
 * silent are DESIGN.md R#1..R#42.
 *
 * Conventions
 *  - Pointers marked (dev) are device memory on the handle's device; (host)
 *    are host memory.  Caller-owned unless stated otherwise.
 *  - `stream` is a cudaStream_t passed as an opaque pointer (NULL = the
 *    legacy default stream).  reset / step / observe / sample_actions /
 *    stats only ENQUEUE work and return; results are valid once that stream
 *    has reached them.  export / import / step_host synchronise.
 *  - Errors: every function returning navix_status validates its host-side
 *    arguments first; on failure it returns a non-zero status, enqueues
 *    nothing, and sets a thread-local message readable with
 *    navix_last_error().  Kernel launch failures return NAVIX_E_CUDA;
 *    asynchronous device faults surface at the caller's next synchronisation.
 *    Invalid ACTION VALUES are not errors: they are no-ops on the device
 *    (R#15), except Dynamic-Obstacles where actions >= 3 act as 0 (R#7).
 *  - No allocation happens on the reset/step path.
 */
#ifndef NAVIX_H_
#define NAVIX_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NAVIX_API __attribute__((visibility("default")))
#else
#define NAVIX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct navix_env navix_env; /* opaque handle: config + state buffers */

typedef enum {
  NAVIX_OK = 0,
  NAVIX_E_UNKNOWN_ENV = 1,  /* env id not in Table 9 / not parsed */
  NAVIX_E_INVALID_ARG = 2,  /* null pointer, bad count, bad shard range, bad record */
  NAVIX_E_CUDA = 3,         /* a CUDA runtime call or kernel launch failed */
  NAVIX_E_NOMEM = 4,        /* device or pinned allocation failed */
  NAVIX_E_UNSUPPORTED = 5   /* a parsed id this build has no kernel for (grids > 24x24; none in Table 9) */
} navix_status;

/* Families of Table 9 with a kernel in this build. */
enum {
  NAVIX_FAMILY_EMPTY = 0,
  NAVIX_FAMILY_DOORKEY = 1,
  NAVIX_FAMILY_DYNOBS = 2,
  NAVIX_FAMILY_KEYCORRIDOR = 3,
  NAVIX_FAMILY_LAVAGAP = 4,
  NAVIX_FAMILY_EMPTY_RANDOM = 5,
  NAVIX_FAMILY_DISTSHIFT = 6,
  NAVIX_FAMILY_CROSSING = 7,
  NAVIX_FAMILY_GOTODOOR = 8,
  NAVIX_FAMILY_FOURROOMS = 9
};

/* Reward modes (R#1/R#3): MINIGRID = legacy 1 - 0.9*sc/T on success,
 * 0 on lava (the BASELINE default); NAVIX = Markovian +1 / -1 (Table 6). */
enum { NAVIX_REWARD_MINIGRID = 0, NAVIX_REWARD_NAVIX = 1 };

/* Static description of an env id (the tuple M = (h, w, T, O, A, ...) of
 * §3.2.1). */
typedef struct {
  int32_t height, width;   /* grid size h, w (Table 9) */
  int32_t view;            /* 7: egocentric view size R (R#14) */
  int32_t n_actions;       /* |A|: 7, or 3 for Dynamic-Obstacles (R#7) */
  int32_t max_steps;       /* T (R#16) */
  int32_t obs_bytes;       /* 147 = 7*7*3, uint8 [vi][vj][channel] (R#10, R#11); 49 with
                            NAVIX_OBS_CATEGORICAL (navix_set_observation) */
  int32_t family;          /* NAVIX_FAMILY_* */
  int32_t n_obstacles;     /* Dynamic-Obstacles balls (R#6), else 0 */
  int32_t export_bytes;    /* canonical per-env record size, see navix_state_export */
} navix_spec;

/* Parse an id such as "Navix-DoorKey-8x8-v0", "MiniGrid-DoorKey-8x8-v0" or
 * "DoorKey-8x8" (Code 1 P:254).  Host only; no CUDA call.
 * Returns NAVIX_E_UNKNOWN_ENV for ids outside Table 8 / Table 9 (P:858-893,
 * P:908-965) and MiniGrid's Dynamic-Obstacles-Random / LavaCrossing spellings
 * (R#35, R#40).  Both tables' spellings are accepted: "LavaGapS7" (Table 8) and
 * "LavaGap-S7" (Table 9); "SimpleCrossingS9N1" (Table 8: wall rivers) and
 * "Crossings-S9N1" (Table 9, reward R_2: lava rivers, = MiniGrid's
 * "LavaCrossingS9N1").  Every Table 8 / Table 9 id has a kernel. */
NAVIX_API navix_status navix_spec_of(const char* env_id, navix_spec* out);

/* Bytes of device state for `num_envs` envs of `env_id` (for a caller-owned
 * state buffer passed to navix_create_shard); 0 if the id/count is invalid. */
NAVIX_API size_t navix_state_bytes(const char* env_id, int64_t num_envs);

/* Shorthand for navix_create_shard(env_id, num_envs, 0, num_envs, seed,
 * <current device>, NULL, NAVIX_REWARD_MINIGRID, out). */
NAVIX_API navix_status navix_create(const char* env_id, int64_t num_envs, uint64_t seed, navix_env** out);

/* Create a handle over the global env indices [env_begin, env_begin+num_envs_local)
 * of a batch of num_envs_total (multi-GPU sharding: every RNG counter uses the
 * GLOBAL index, so shards concatenate to the unsharded batch bit-for-bit, R#20).
 *  seed        64-bit Philox key of the level and obstacle streams (R#20).
 *  device      CUDA device ordinal that will own the state.
 *  state_dev   (dev, nullable) caller-owned buffer of navix_state_bytes(env_id,
 *              num_envs_local) bytes, 256-byte aligned; NULL = the library
 *              cudaMallocs it and frees it in navix_destroy.
 * No kernel runs; navix_reset (or navix_state_import) must precede the first
 * step / rollout / observe (else NAVIX_E_INVALID_ARG). */
NAVIX_API navix_status navix_create_shard(const char* env_id, int64_t num_envs_total, int64_t env_begin,
                                int64_t num_envs_local, uint64_t seed, int device, void* state_dev,
                                int reward_mode, navix_env** out);

/* reset(key) for every env: episode 0, level generated from
 * Philox(seed; env, 0, 0, block), statistics zeroed.
 *  obs  (dev) uint8[n][7][7][3]: the FIRST observation (any alignment; a
 *        16-byte aligned buffer enables the per-tile TMA bulk store). */
NAVIX_API navix_status navix_reset(navix_env* h, uint8_t* obs, void* stream);

/* reset(key) with a new key (Code 1 P:264): the handle's seed becomes
 * `seed` for this and every later level / obstacle draw, then navix_reset.
 * Equivalent to destroying the handle and creating it with `seed`.
 * Kernel arguments are passed by value: a CUDA graph captured before this
 * call replays the old setting; recapture graphs after calling it. */
NAVIX_API navix_status navix_reset_seed(navix_env* h, uint64_t seed, uint8_t* obs, void* stream);

/* One step of every env with next-step auto-reset (R#18):
 *  actions     (dev) uint8[n]
 *  obs         (dev) uint8[n][7][7][3] (16-byte aligned: bulk-store fast path)
 *  reward      (dev) float[n]     (R#1/R#2/R#3, R_3 = -1 on collision R#4)
 *  terminated  (dev) uint8[n]     0/1 (event: goal, lava, collision, KeyCorridor ball,
 *                                  GoToDoor toggle / done, R#37)
 *  truncated   (dev) uint8[n]     0/1 (step_count reached T without an event, R#17)
 * An env whose previous step ended ignores its action, starts its next
 * episode and returns that episode's first observation with reward 0 and
 * both flags 0.  Episode statistics are accumulated on terminal steps. */
NAVIX_API navix_status navix_step(navix_env* h, const uint8_t* actions, uint8_t* obs, float* reward,
                        uint8_t* terminated, uint8_t* truncated, void* stream);

/* K consecutive steps in ONE launch (the analogue of the
 * paper's lax.scan over the step, Code 2-3 P:603-660): bit-identical to K
 * navix_step calls with actions[t], while the environment state stays on chip
 * between the steps (only actions in, observations / rewards / flags out).
 *  actions     (dev) uint8[steps][n]
 *  obs         (dev) uint8[steps][n][7][7][3]   (n % 16 == 0 and a 16-byte
 *              aligned base enable the per-tile TMA bulk store)
 *  reward      (dev) float[steps][n];  terminated, truncated (dev) uint8[steps][n] */
NAVIX_API navix_status navix_rollout(navix_env* h, const uint8_t* actions, int64_t steps, uint8_t* obs,
                                     float* reward, uint8_t* terminated, uint8_t* truncated, void* stream);

/* navix_rollout with the uniform random policy drawn inside the kernel
 * (SURVEY §8f row f1): the action of env i at step t is the one
 * navix_sample_actions(action_seed, t0 + t) writes (Philox key action_seed,
 * counter (global env index, t0 + t, 2 << 16, 0), word 0, bounded by
 * n_actions), so the results equal navix_rollout on those sampled actions.
 * No action buffer is read.  Outputs as navix_rollout. */
NAVIX_API navix_status navix_rollout_random(navix_env* h, uint64_t action_seed, int64_t t0, int64_t steps,
                                            uint8_t* obs, float* reward, uint8_t* terminated, uint8_t* truncated,
                                            void* stream);

/* Reward composition (Table 6 `time_cost`, `action_cost`; Code 4 `compose`,
 * P:673-680; R#31): every later step adds -time_cost, and
 * -action_cost unless the action is done (6), to the event reward, in binary32
 * in that order.  Auto-reset calls still return 0.  Both >= 0; 0 disables.
 * Host only, takes effect for subsequently enqueued steps.
 * Kernel arguments are passed by value: a CUDA graph captured before this
 * call replays the old setting; recapture graphs after calling it. */
NAVIX_API navix_status navix_set_reward_costs(navix_env* h, float time_cost, float action_cost);

/* Reward / termination function selection (Table 6 / Table 7, P:566-589;
 * Code 4 `compose`; R#42).  Every family's events are exclusive:
 *   NAVIX_EVENT_GOAL    (1) the goal / success event: on_goal_reached, and the
 *                           family's success (KeyCorridor ball pickup, GoToDoor
 *                           door: on_door_done in the navix reward mode)
 *   NAVIX_EVENT_LAVA    (2) on_lava_fall
 *   NAVIX_EVENT_FAILURE (4) Dynamic-Obstacles collision (R_3), GoToDoor's
 *                           toggle / done away from the target ([MG])
 * reward_events selects the events that pay their reward (else 0; 0 = the
 * `free` reward function); termination_events the events that end the
 * episode (0 = `free`: only truncation ends episodes; an event that does not
 * terminate is not counted in the statistics).  Default 7 / 7 (Table 9's
 * R_1 / R_2 / R_3).  Composes with navix_set_reward_costs.  Host only.
 * Kernel arguments are passed by value: a CUDA graph captured before this
 * call replays the old setting; recapture graphs after calling it. */
enum { NAVIX_EVENT_GOAL = 1, NAVIX_EVENT_LAVA = 2, NAVIX_EVENT_FAILURE = 4 };
NAVIX_API navix_status navix_set_event_functions(navix_env* h, uint32_t reward_events, uint32_t termination_events);

/* Small batches: a step or rollout of at most max_envs envs
 * runs the multi-lane-per-env kernels (8 lanes share an env and split its
 * observation by view column), larger ones the one-thread-per-env kernels.
 * Results are bit-identical either way; only the latency differs.  Defaults:
 * 2048 envs for steps (NAVIX_DEFAULT_WIDE_MAX, environment variable
 * NAVIX_WIDE_MAX) and 4096 for rollouts (NAVIX_DEFAULT_WIDE_MAX_ROLLOUT,
 * NAVIX_WIDE_MAX_ROLLOUT); this call sets both; 0 disables.  Grids up to 8
 * wide except GoToDoor (and KeyCorridor steps).  Host only; graphs captured earlier keep the old
 * choice. */
NAVIX_API navix_status navix_set_small_batch_threshold(navix_env* h, int64_t max_envs);

/* Observation kinds (Table 5; R#41).  SYMBOLIC (the
 * default): first-person records uint8[7][7][3] = 147 B (symbolic_first_person)
 * and full grids uint8[W][H][3] (symbolic).  CATEGORICAL: the entity type
 * alone, uint8[7][7] = 49 B (categorical_first_person) and uint8[W][H]
 * (categorical); unseen view cells are 0.  The kind applies to every obs
 * output enqueued afterwards (reset, step, step_host, rollout, observe,
 * observe_full); size obs buffers accordingly.  Host only.
 * Kernel arguments are passed by value: a CUDA graph captured before this
 * call replays the old setting; recapture graphs after calling it. */
enum { NAVIX_OBS_SYMBOLIC = 0, NAVIX_OBS_CATEGORICAL = 1 };
NAVIX_API navix_status navix_set_observation(navix_env* h, int kind);

/* Table 5 `symbolic` full-grid observation, MiniGrid's
 * FullyObsWrapper: out (dev) uint8[n][width][height][3] ([x][y][c]), every
 * cell encoded (type, colour, state) and the agent cell (10, 0, dir) (R#32);
 * uint8[n][width][height] (types, agent 10) with NAVIX_OBS_CATEGORICAL. */
NAVIX_API navix_status navix_observe_full(navix_env* h, uint8_t* out, void* stream);

/* The current observation of every env without stepping (O: S -> O, Table 3). */
NAVIX_API navix_status navix_observe(navix_env* h, uint8_t* obs, void* stream);

/* GoToDoor's mission (Table 6 / 7 `on_door_done`: "the colour specified in
 * the mission"; R#37): out (dev) uint8[n] = MiniGrid colour
 * index (0 red .. 5 grey) of each env's target door, for the current
 * episode.  NAVIX_E_INVALID_ARG for other families. */
NAVIX_API navix_status navix_observe_mission(navix_env* h, uint8_t* out, void* stream);

/* The random policy of the bench (R#20, domain 2):
 * out[t][i] = bounded(word0(Philox(ctr=(env_begin+i, t0+t, 2<<16, 0),
 * key=action_seed)), n_actions).   out (dev) uint8[steps][n]. */
NAVIX_API navix_status navix_sample_actions(navix_env* h, uint64_t action_seed, int64_t t0, int64_t steps,
                                  uint8_t* out, void* stream);

/* End-to-end step through host buffers: copies actions host->device,
 * steps, copies obs/reward/flags device->host, and synchronises `stream`.
 * All five pointers are (host) arrays sized as in navix_step; pinned memory
 * is fastest.  Library-owned device staging is allocated on first use. */
NAVIX_API navix_status navix_step_host(navix_env* h, const uint8_t* actions, uint8_t* obs, float* reward,
                             uint8_t* terminated, uint8_t* truncated, void* stream);

/* Episode statistics of this shard since the last reset (info i_{t+1},
 * P:238): out8 (dev) int64[8] = {episodes, sum of lengths, n_success,
 * sum of step counts at success, n_lava, n_failure (Dynamic-Obstacles
 * collision; GoToDoor toggle or done away from the target), n_truncated,
 * generator failures}.  Exact integers: summing over shards (an all-reduce)
 * gives the unsharded values. */
NAVIX_API navix_status navix_stats(navix_env* h, int64_t* out8, void* stream);

/* Canonical state record per env (parity / checkpoint), little endian:
 *   H*W cells as MiniGrid (type, colour, state), row-major y outer, x inner;
 *   agent x, y, dir; carry (type, colour), (1, 0) = nothing;
 *   step_count u16; episode u32; prev_done u8;
 *   Dynamic-Obstacles: n_obstacles x (x, y) in creation order;
 *   GoToDoor: the target door's (x, y).
 * export: synchronises the device, writes n*export_bytes into `host`.
 * import: validates every record (closed wall border, agent on a walkable
 * interior cell, legal codes, balls consistent; GoToDoor: any border, agent
 * anywhere walkable, target inside the grid) before touching the device. */
NAVIX_API navix_status navix_state_export(navix_env* h, void* host, size_t cap, size_t* written);
NAVIX_API navix_status navix_state_import(navix_env* h, const void* host, size_t n_bytes);

/* out4 = {num_envs_local, env_begin, num_envs_total, device}. */
NAVIX_API navix_status navix_info(navix_env* h, int64_t* out4);

NAVIX_API void navix_destroy(navix_env* h);

/* Thread-local text of the last failure on this thread ("" if none). */
NAVIX_API const char* navix_last_error(void);

/* Build provenance: the 16-hex-digit hash of every source file and compiler
 * flag this library was compiled from (paper_2407_19396_b200/build.py
 * source_hash()); the tests compare it with the checked-out tree, so a stale
 * prebuilt libnavix.so fails loudly instead of being tested.  Host only. */
NAVIX_API const char* navix_build_id(void);

#ifdef __cplusplus
}
#endif
#endif /* NAVIX_H_ */
