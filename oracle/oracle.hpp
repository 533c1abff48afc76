// oracle/oracle.hpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU oracle of the batched MiniGrid step that
// NAVIX (arXiv 2407.19396) re-implements.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.  It shares
// no code, header, table or constant with paper_2407_19396_b200/csrc (the CUDA
// product path), and the product path never loads it.
//
// Citations: "P:L" = /root/reference/PAPER.md line L; "S:L" = SPEC.md line L;
// "[MG]" = an upstream MiniGrid rule the paper claims to reproduce exactly
// ("NAVIX matches the original MiniGrid suite in terms of
// environments, observations, state transitions, rewards, and actions");
// "R#n" = reading n in DESIGN.md "Readings of the paper".
//
// Data model (deliberately unlike the GPU's packed uint8 planes): an
// object grid of std::optional<Obj> indexed [j*width+i] exactly like
// MiniGrid's Grid, the agent as separate fields, and literal transcriptions of
// Grid.slice, Grid.rotate_left, Grid.process_vis and Grid.encode.
#pragma once
#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace oracle {

// [MG] OBJECT_TO_IDX / COLOR_TO_IDX / STATE_TO_IDX (minigrid.core.constants).
enum : uint8_t {
  T_UNSEEN = 0, T_EMPTY = 1, T_WALL = 2, T_FLOOR = 3, T_DOOR = 4, T_KEY = 5,
  T_BALL = 6, T_BOX = 7, T_GOAL = 8, T_LAVA = 9, T_AGENT = 10
};
enum : uint8_t { C_RED = 0, C_GREEN = 1, C_BLUE = 2, C_PURPLE = 3, C_YELLOW = 4, C_GREY = 5 };
// [MG] Actions: left, right, forward, pickup, drop, toggle, done.
enum : int { A_LEFT = 0, A_RIGHT = 1, A_FORWARD = 2, A_PICKUP = 3, A_DROP = 4, A_TOGGLE = 5, A_DONE = 6 };

// Families of Table 9 implemented by the oracle.
enum Family : int { F_EMPTY = 0, F_DOORKEY = 1, F_DYNOBS = 2, F_KEYCORRIDOR = 3, F_LAVAGAP = 4, F_EMPTY_RANDOM = 5,
                    F_DISTSHIFT = 6, F_CROSSING = 7, F_GOTODOOR = 8,
                    F_FOURROOMS = 9 };

// One MiniGrid WorldObj.  `tag` is test-only bookkeeping (rotation pin P6).
struct Obj {
  uint8_t type = T_EMPTY;
  uint8_t color = 0;
  bool is_open = false;
  bool is_locked = false;
  int tag = 0;

  // [MG] WorldObj.can_overlap: Goal, Lava, Floor -> True; Door -> is_open.
  bool can_overlap() const;
  // [MG] WorldObj.see_behind: Wall -> False; Door -> is_open; else True.
  bool see_behind() const;
  // [MG] Key, Ball, Box -> can_pickup.
  bool can_pickup() const;
  // [MG] WorldObj.encode -> (OBJECT_TO_IDX, COLOR_TO_IDX, state);
  // Door state: 0 open, 1 closed, 2 locked.
  void encode(uint8_t out[3]) const;
};
using Cell = std::optional<Obj>;

Obj make_wall();
Obj make_goal();
Obj make_lava();
Obj make_key(uint8_t color);
Obj make_ball(uint8_t color);
Obj make_door(uint8_t color, bool is_locked);

// [MG] minigrid.core.grid.Grid, transcribed literally.
struct Grid {
  int width, height;
  std::vector<Cell> grid;  // index j*width + i, as in [MG]
  Grid(int w, int h);
  const Cell& get(int i, int j) const;
  void set(int i, int j, const Cell& v);
  void horz_wall(int x, int y, int length, const Obj& o);
  void vert_wall(int x, int y, int length, const Obj& o);
  void wall_rect(int x, int y, int w, int h);
  Grid slice(int topX, int topY, int w, int h) const;
  Grid rotate_left() const;
  // returns mask[i*height + j] ([MG] np array of shape (width, height))
  std::vector<uint8_t> process_vis(int agent_x, int agent_y) const;
  // out[(i*height + j)*3 + c] ([MG] array of shape (width, height, 3))
  void encode(const std::vector<uint8_t>& vis_mask, uint8_t* out) const;
};

// Static per-env-id configuration (P:209 tuple M=(h,w,T,...)), see R#16.
struct Spec {
  Family family;
  int height, width;
  int max_steps;      // T
  int n_actions;      // |A|
  int size;           // S for Empty/DoorKey/DynObs/LavaGap
  int room_size;      // KeyCorridor s
  int num_rows;       // KeyCorridor R
  int n_obstacles;    // DynObs
  int strip2_row;     // DistShift
  int n_crossings;    // SimpleCrossing N
  bool lava_obstacle;  // Crossings: lava rivers (Table 9 R_2, LavaCrossing) instead of walls
  bool random_start;  // Dynamic-Obstacles-Random: place_agent() instead of (1,1) east
};
// Parses "Navix-DoorKey-8x8-v0" / "MiniGrid-…" / bare ids. false if unknown.
bool parse_env_id(const std::string& env_id, Spec* out);

// Philox4x32-10 (Salmon et al., SC'11), written out round by round.
void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
// Lemire multiply-high without rejection (R#21).
uint32_t bounded(uint32_t u, uint32_t n);

// A stream of 32-bit draws: draw k = word (k mod 4) of the Philox block with
// counter (c0, c1, c2, k/4) under key (seed lo, seed hi).  (R#20.)
struct DrawStream {
  uint32_t key[2];
  uint32_t c0, c1, c2;
  uint64_t k = 0;
  DrawStream(uint64_t seed, uint32_t c0_, uint32_t c1_, uint32_t c2_);
  uint32_t next();
  uint32_t next_bounded(uint32_t n) { return bounded(next(), n); }
};

enum RewardMode : int { RM_MINIGRID = 0, RM_NAVIX = 1 };

struct StepOut {
  float reward = 0.f;
  bool terminated = false, truncated = false;
};

// One MiniGrid environment instance (MiniGridEnv + the per-family subclass).
struct Env {
  Spec spec;
  int reward_mode = RM_MINIGRID;
  float time_cost = 0.f, action_cost = 0.f;  // Table 6 time_cost / action_cost (R#31)
  // Table 6 / Table 7 selection (R#42): which events pay their reward and
  // which end the episode; bit 0 the goal / success event, bit 1 lava, bit 2
  // failure (collision, GoToDoor toggle / done away).  0 = `free`.
  uint32_t reward_events = 7, termination_events = 7;
  uint64_t seed = 0;
  uint32_t global_index = 0;  // c0 of every Philox counter (shard invariance)
  Grid grid{1, 1};
  int agent_x = 0, agent_y = 0, agent_dir = 0;
  int target_x = 0, target_y = 0;  // GoToDoor: [MG] target_pos
  Cell carrying;
  int step_count = 0;
  uint32_t episode = 0;
  bool prev_done = false;
  std::vector<std::pair<int, int>> obstacles;  // DynObs balls, creation order
  // per-env episode statistics contributions (summed by the handle)
  int64_t stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  void generate();  // P0 for episode `episode` (levels.cpp)
  StepOut step(int action);
  void gen_obs(uint8_t* out147) const;
  void gen_full_obs(uint8_t* out) const;  // Table 5 `symbolic`, [x][y][c] (R#32)
  std::pair<int, int> front_pos() const;
};

// Stats slots.
enum { ST_EPISODES = 0, ST_SUM_LEN, ST_SUCCESS, ST_SUM_SUCCESS_STEP, ST_LAVA, ST_FAILURE, ST_TRUNCATED, ST_GEN_FAIL };

// Canonical export record size per env.
int export_bytes_per_env(const Spec& s);
void export_env(const Env& e, uint8_t* out);
bool import_env(Env& e, const uint8_t* in);

// Success reward of reward mode `mode` at step count sc with horizon T (R#1, R#2).
float success_reward(int mode, int sc, int T);

}  // namespace oracle
