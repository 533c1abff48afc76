// layout.h — internal data layout of libnavix (host + device).
//
// HBM state of one handle (one shard), a single allocation:
//   grid    u64 [n_tiles][H*RW][TILE] row y of env (tile, slot) as RW planes
//                                     (RW = 1 up to width 8, 2 up to 16): byte
//                                     x % 8 of plane y*RW + x/8 = cell (x, y);
//                                     cells x >= W are 0
//   agent   u64 [n_pad]               agent record (below)
//   episode u32 [n_pad]               episode counter (counter word c1, R#20)
//   balls   u64 [n_pad]               Dynamic-Obstacles: byte b = ball_code(W, x, y) of ball b (<= 8)
//   stats   u64 [NSLOT][8]            striped int64 episode statistics
//   sched   u32 [8 + 4 n_tiles]       persistent step kernel tile scheduler (+ reset-first tile lists)
// n_pad = num_envs rounded up to TILE.  The struct-of-arrays "row plane"
// layout makes every warp load of a grid row one contiguous 256-byte segment
// and lets the kernel fetch a whole world row with one 64-bit load.
//
// Cell byte: bit 7 = opaque (wall, closed door, locked door: see_behind is
// False), bits 4-6 = MiniGrid colour, bits 0-3 = kind:
//   1 empty, 2 wall, 3 floor, 4 open door, 5 key, 6 ball, 7 box, 8 goal,
//   9 lava, 11 closed door, 12 locked door.   0 = outside the grid.
// obs type = kind >= 11 ? 4 : kind; obs state = kind >= 11 ? kind - 10 : 0;
// obs colour = bits 4-6.  Dynamic-Obstacles balls are NOT stored in the HBM
// grid (it holds the static layout); they are overlaid from `balls` in SMEM.
//
// Agent record (u64, little endian bytes): 0 x, 1 y, 2 dir, 3 carry (cell
// byte of the carried object, 0x01 = nothing), 4-5 step_count, 6 flags
// (bit 0 prev_done; bit 1 static-layout families: the HBM grid holds the
// family's template; bit 2 DoorKey / LavaGap / Crossings: the visibility
// table applies, keyed by byte 7 for DoorKey; GoToDoor: a generated room
// with its doors still closed, so the view needs no out-of-grid walls), 7 GoToDoor target door
// (x << 4) | y, DoorKey (split << 4) | door_y of its generated layout.
#pragma once
#include <cstdint>

namespace navix {

constexpr int TILE = 128;   // envs per CTA (one thread per env)
#ifndef NAVIX_DEFAULT_WIDE_MAX
#define NAVIX_DEFAULT_WIDE_MAX 2048  // small-batch kernel up to this many envs (measured)
#endif
#ifndef NAVIX_DEFAULT_WIDE_MAX_ROLLOUT
#define NAVIX_DEFAULT_WIDE_MAX_ROLLOUT 4096  // the same for rollouts (measured)
#endif
constexpr int NSLOT = 512;  // stats stripes (atomics spread over 512 x 64 B)
constexpr int OBS_BYTES = 147;
// Observation kinds (Table 5, R#41): the first-person record is
// 147 B (symbolic, [vi][vj][type, colour, state]) or 49 B (categorical,
// [vi][vj] entity type); the full grid is 3*W*H or W*H bytes, [x][y](c).
enum ObsKind : int { OBS_SYMBOLIC = 0, OBS_CATEGORICAL = 1 };
__host__ __device__ constexpr int obs_record_bytes(int kind) { return kind == OBS_CATEGORICAL ? 49 : OBS_BYTES; }

enum Kind : uint8_t {
  K_OOB = 0, K_EMPTY = 1, K_WALL = 2, K_FLOOR = 3, K_DOOR_OPEN = 4, K_KEY = 5, K_BALL = 6,
  K_BOX = 7, K_GOAL = 8, K_LAVA = 9, K_DOOR_CLOSED = 11, K_DOOR_LOCKED = 12
};
constexpr uint8_t OPAQUE_BIT = 0x80;

__host__ __device__ constexpr uint8_t make_cell(uint8_t kind, uint8_t colour) {
  return (uint8_t)(((kind == K_WALL || kind == K_DOOR_CLOSED || kind == K_DOOR_LOCKED) ? OPAQUE_BIT : 0) |
                   ((colour & 7) << 4) | kind);
}
// MiniGrid colours
constexpr uint8_t COL_RED = 0, COL_GREEN = 1, COL_BLUE = 2, COL_PURPLE = 3, COL_YELLOW = 4, COL_GREY = 5;
constexpr uint8_t CELL_EMPTY = make_cell(K_EMPTY, 0);
constexpr uint8_t CELL_WALL = make_cell(K_WALL, COL_GREY);
constexpr uint8_t CELL_GOAL = make_cell(K_GOAL, COL_GREEN);
constexpr uint8_t CELL_LAVA = make_cell(K_LAVA, COL_RED);

enum Family : int { FAM_EMPTY = 0, FAM_DOORKEY = 1, FAM_DYNOBS = 2, FAM_KEYCORRIDOR = 3, FAM_LAVAGAP = 4,
                    FAM_EMPTY_RANDOM = 5, FAM_DISTSHIFT1 = 6, FAM_DISTSHIFT2 = 7, FAM_CROSSING = 8,
                    FAM_GOTODOOR = 9, FAM_FOURROOMS = 10 };

struct EnvConfig {
  int family;
  int height, width;
  int max_steps;
  int n_actions;
  int n_obstacles;
  int room_size, num_rows;  // KeyCorridor
  int gen_param;            // Crossing: number of crossings N | CROSSING_LAVA
};
constexpr int CROSSING_LAVA = 0x100;  // gen_param bit: lava rivers (Table 9 Crossings / LavaCrossing, R#35)

// Byte offsets of the arrays inside one state allocation.
struct StateLayout {
  int64_t n_pad, n_tiles;
  size_t grid_off, agent_off, episode_off, balls_off, stats_off, sched_off, total;
};

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Dynamic-Obstacles ball byte (byte b of the balls word = ball b, 0 = none):
// on grids up to 8 wide the transition's bitboard index 8 y + x, on wider
// grids (x << 4) | y.  Interior positions never encode to 0.
__host__ __device__ constexpr uint32_t ball_code(int width, int x, int y) {
  return width <= 8 ? (uint32_t)(8 * y + x) : (uint32_t)((x << 4) | y);
}
__host__ __device__ constexpr int ball_x(int width, uint32_t p) { return width <= 8 ? (int)(p & 7) : (int)(p >> 4); }
__host__ __device__ constexpr int ball_y(int width, uint32_t p) { return width <= 8 ? (int)(p >> 3) : (int)(p & 15); }

// u64 planes per grid row: 8-byte rows up to width 8, 16-byte rows up to 16 (row f2)
__host__ __device__ constexpr int row_planes(int width) { return (width + 7) / 8; }

inline StateLayout make_layout(const EnvConfig& c, int64_t n) {
  StateLayout L{};
  L.n_tiles = (n + TILE - 1) / TILE;
  L.n_pad = L.n_tiles * TILE;
  size_t off = 0;
  L.grid_off = off;
  off = align_up(off + (size_t)L.n_pad * c.height * row_planes(c.width) * 8, 256);
  L.agent_off = off;
  off = align_up(off + (size_t)L.n_pad * 8, 256);
  L.episode_off = off;
  off = align_up(off + (size_t)L.n_pad * 4, 256);
  L.balls_off = off;
  off = align_up(off + (c.family == FAM_DYNOBS ? (size_t)L.n_pad * 8 : 0), 256);
  L.stats_off = off;
  off = align_up(off + (size_t)NSLOT * 8 * 8, 256);
  // scheduler: 8 words ([0] ticket, [1] CTAs done, [2] step epoch, [3..4]
  // list counts by epoch parity), then by epoch parity: per tile the epoch
  // stamp of "has envs to reset at that step", and the list of those tiles
  L.sched_off = off;
  off = align_up(off + (8 + 4 * (size_t)L.n_tiles) * sizeof(unsigned int), 256);
  L.total = off;
  return L;
}

// Tile-local env le <-> state slot (see step_kernel.cuh): warp w lane l owns
// env 4*l + w and slot 32*w + l.
__host__ __device__ constexpr int slot_of_env(int le) { return (le & 3) * 32 + (le >> 2); }
__host__ __device__ constexpr int env_of_slot(int slot) { return 4 * (slot & 31) + (slot >> 5); }

// Kernel arguments (by value).
struct KernelArgs {
  uint64_t* grid;
  uint64_t* agent;
  uint32_t* episode;
  uint64_t* balls;
  unsigned long long* stats;
  unsigned int* sched;  // persistent tile scheduler {next tile, CTAs done}
  const uint8_t* actions;
  uint8_t* obs;
  float* reward;
  uint8_t* terminated;
  uint8_t* truncated;
  int64_t n;            // local envs
  uint32_t env_begin;   // global index of local env 0 (Philox counter word c0)
  uint32_t key_lo, key_hi;
  int reward_mode;
  float time_cost, action_cost;  // Table 6 time_cost / action_cost, composed with the event reward (R#31)
  int bulk_obs;         // 1: obs base is 16-B aligned -> cp.async.bulk store of full tiles
  int bulk_act;         // 1: actions base is 16-B aligned -> cp.async.bulk load of full tiles
  int64_t rollout_steps;  // K of navix_rollout
  int gen_param;        // EnvConfig::gen_param (runtime level-generator parameter)
  int obs_kind;         // ObsKind of the obs outputs
  uint32_t reward_events, termination_events;  // Table 6 / 7 selection (R#42): bit 0 success, 1 lava, 2 failure
  // rollout with actions == nullptr: in-kernel uniform random policy, the
  // navix_sample_actions stream (key act_key, counter (env, act_t0 + t, 2 << 16, 0))
  uint32_t act_key_lo, act_key_hi, act_t0;
  int64_t wide_max;     // steps of at most this many envs run navix_step_wide (small batches)
  int64_t wide_max_rollout;  // rollouts of at most this many envs run navix_rollout_wide
};

enum Mode : int { MODE_STEP = 0, MODE_RESET = 1, MODE_OBSERVE = 2, MODE_ROLLOUT = 3, MODE_FULL_OBS = 4,
                  MODE_OBS_TABLE = 5 /* build the Dynamic-Obstacles observation table (step_kernel.cuh) */ };

}  // namespace navix
