// oracle/minigrid.cpp — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
//
// Literal transcription of upstream MiniGrid's world objects, Grid and
// MiniGridEnv.step / gen_obs, which the paper claims to match exactly
// (P:114).  Systems of Table 3: Intervention I,
// Transition mu (DynObs only), Observation O = symbolic_first_person
// (Table 5), Reward R (Eq. 1 P:216 / P:223; Table 6 P:571-572;
// Table 9 caption P:971-974), Termination gamma (Table 7).
#include <algorithm>
#include <cassert>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include <cstdlib>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- objects
bool Obj::can_overlap() const {
  switch (type) {
    case T_GOAL: case T_LAVA: case T_FLOOR: return true;
    case T_DOOR: return is_open;
    default: return false;
  }
}
bool Obj::see_behind() const {
  switch (type) {
    case T_WALL: return false;
    case T_DOOR: return is_open;
    default: return true;
  }
}
bool Obj::can_pickup() const { return type == T_KEY || type == T_BALL || type == T_BOX; }
void Obj::encode(uint8_t out[3]) const {
  out[0] = type;
  out[1] = color;
  uint8_t state = 0;
  if (type == T_DOOR) {
    // [MG] Door.encode: open 0, locked 2, closed 1
    if (is_open) state = 0;
    else if (is_locked) state = 2;
    else state = 1;
  }
  out[2] = state;
}

static Obj mk(uint8_t t, uint8_t c) { Obj o; o.type = t; o.color = c; return o; }
Obj make_wall() { return mk(T_WALL, C_GREY); }    // [MG] Wall(color="grey")
Obj make_goal() { return mk(T_GOAL, C_GREEN); }   // [MG] Goal: green
Obj make_lava() { return mk(T_LAVA, C_RED); }     // [MG] Lava: red
Obj make_key(uint8_t c) { return mk(T_KEY, c); }
Obj make_ball(uint8_t c) { return mk(T_BALL, c); }
Obj make_door(uint8_t c, bool locked) {
  Obj o = mk(T_DOOR, c);
  o.is_locked = locked;
  o.is_open = false;
  return o;
}

// ---------------------------------------------------------------- Grid
Grid::Grid(int w, int h) : width(w), height(h), grid((size_t)w * h) {}

const Cell& Grid::get(int i, int j) const {
  if (i < 0 || i >= width || j < 0 || j >= height) throw std::out_of_range("Grid.get");
  return grid[(size_t)j * width + i];
}
void Grid::set(int i, int j, const Cell& v) {
  if (i < 0 || i >= width || j < 0 || j >= height) throw std::out_of_range("Grid.set");
  grid[(size_t)j * width + i] = v;
}
void Grid::horz_wall(int x, int y, int length, const Obj& o) {
  if (length < 0) length = width - x;
  for (int i = 0; i < length; ++i) set(x + i, y, o);
}
void Grid::vert_wall(int x, int y, int length, const Obj& o) {
  if (length < 0) length = height - y;
  for (int j = 0; j < length; ++j) set(x, y + j, o);
}
void Grid::wall_rect(int x, int y, int w, int h) {
  horz_wall(x, y, w, make_wall());
  horz_wall(x, y + h - 1, w, make_wall());
  vert_wall(x, y, h, make_wall());
  vert_wall(x + w - 1, y, h, make_wall());
}

// [MG] Grid.slice: out-of-grid cells become Wall().
Grid Grid::slice(int topX, int topY, int w, int h) const {
  Grid g(w, h);
  for (int j = 0; j < h; ++j) {
    for (int i = 0; i < w; ++i) {
      int x = topX + i, y = topY + j;
      Cell v;
      if (0 <= x && x < width && 0 <= y && y < height) v = get(x, y);
      else v = make_wall();
      g.set(i, j, v);
    }
  }
  return g;
}

// [MG] Grid.rotate_left: grid.set(j, grid.height - 1 - i, self.get(i, j)).
Grid Grid::rotate_left() const {
  Grid g(height, width);
  for (int i = 0; i < width; ++i)
    for (int j = 0; j < height; ++j) g.set(j, g.height - 1 - i, get(i, j));
  return g;
}

// [MG] Grid.process_vis, both per-row loops exactly as upstream.
std::vector<uint8_t> Grid::process_vis(int agent_x, int agent_y) const {
  std::vector<uint8_t> mask((size_t)width * height, 0);
  auto M = [&](int i, int j) -> uint8_t& { return mask[(size_t)i * height + j]; };
  M(agent_x, agent_y) = 1;
  for (int j = height - 1; j >= 0; --j) {
    for (int i = 0; i < width - 1; ++i) {
      if (!M(i, j)) continue;
      const Cell& cell = get(i, j);
      if (cell && !cell->see_behind()) continue;
      M(i + 1, j) = 1;
      if (j > 0) {
        M(i + 1, j - 1) = 1;
        M(i, j - 1) = 1;
      }
    }
    for (int i = width - 1; i >= 1; --i) {
      if (!M(i, j)) continue;
      const Cell& cell = get(i, j);
      if (cell && !cell->see_behind()) continue;
      M(i - 1, j) = 1;
      if (j > 0) {
        M(i - 1, j - 1) = 1;
        M(i, j - 1) = 1;
      }
    }
  }
  return mask;
}

// [MG] Grid.encode(vis_mask): None -> (empty, 0, 0); invisible -> (0, 0, 0).
void Grid::encode(const std::vector<uint8_t>& vis_mask, uint8_t* out) const {
  for (int i = 0; i < width; ++i) {
    for (int j = 0; j < height; ++j) {
      uint8_t* o = out + ((size_t)i * height + j) * 3;
      o[0] = o[1] = o[2] = 0;
      if (!vis_mask[(size_t)i * height + j]) continue;
      const Cell& v = get(i, j);
      if (!v) { o[0] = T_EMPTY; o[1] = 0; o[2] = 0; }
      else v->encode(o);
    }
  }
}

// ---------------------------------------------------------------- spec
static bool parse_int(const std::string& s, size_t& pos, int* out) {
  size_t b = pos;
  int v = 0;
  while (pos < s.size() && s[pos] >= '0' && s[pos] <= '9') { v = v * 10 + (s[pos] - '0'); ++pos; }
  if (pos == b || pos - b > 3) return false;
  *out = v;
  return true;
}
static bool starts_with(const std::string& s, const std::string& p) { return s.compare(0, p.size(), p) == 0; }

bool parse_env_id(const std::string& id_in, Spec* out) {
  std::string id = id_in;
  if (starts_with(id, "Navix-")) id = id.substr(6);
  else if (starts_with(id, "MiniGrid-")) id = id.substr(9);
  if (id.size() > 3 && id.compare(id.size() - 3, 3, "-v0") == 0) id = id.substr(0, id.size() - 3);
  Spec s{};
  size_t pos = 0;
  auto square = [&](const std::string& prefix, Family f) -> bool {
    if (!starts_with(id, prefix)) return false;
    pos = prefix.size();
    int a, b;
    if (!parse_int(id, pos, &a)) return false;
    if (pos >= id.size() || id[pos] != 'x') return false;
    ++pos;
    if (!parse_int(id, pos, &b)) return false;
    if (pos != id.size() || a != b) return false;
    s.family = f;
    s.size = a;
    s.height = s.width = a;
    return true;
  };
  if (square("Empty-Random-", F_EMPTY_RANDOM)) {
    // [MG] EmptyEnv(size, agent_start_pos=None): random start cell and direction
    if (s.size < 5 || s.size > 16) return false;
    s.max_steps = 4 * s.size * s.size;
    s.n_actions = 7;
  } else if (id == "DistShift1" || id == "DistShift2") {
    // [MG] DistShiftEnv(width=9, height=7, strip2_row=2 / 5) (R#33)
    s.family = F_DISTSHIFT;
    s.width = 9;
    s.height = 7;
    s.strip2_row = id == "DistShift1" ? 2 : 5;
    s.max_steps = 4 * 9 * 7;
    s.n_actions = 7;
  } else if (starts_with(id, "SimpleCrossingS") || starts_with(id, "Crossings-S") ||
             starts_with(id, "LavaCrossingS")) {
    // [MG] CrossingEnv(size, num_crossings, obstacle_type): Table 8's
    // SimpleCrossing ids have wall rivers; Table 9's
    // "Crossings-S9N1" ids carry R_2, read as [MG]'s
    // LavaCrossing, obstacle_type=Lava (R#35)
    s.lava_obstacle = !starts_with(id, "SimpleCrossingS");
    pos = starts_with(id, "SimpleCrossingS") ? 15 : starts_with(id, "LavaCrossingS") ? 13 : 11;
    int S, N;
    if (!parse_int(id, pos, &S)) return false;
    if (pos >= id.size() || id[pos] != 'N') return false;
    ++pos;
    if (!parse_int(id, pos, &N) || pos != id.size()) return false;
    if (S < 5 || S > 16 || S % 2 == 0) return false;  // [MG] asserts odd sizes
    if (N < 1 || N > 2 * ((S - 3) / 2)) return false;   // at most every river
    s.family = F_CROSSING;
    s.size = S;
    s.height = s.width = S;
    s.n_crossings = N;
    s.max_steps = 4 * S * S;  // [MG] CrossingEnv
    s.n_actions = 7;
  } else if (id == "FourRooms") {
    // [MG] FourRoomsEnv at Table 9's 17x17 (MG's default is 19), max_steps 100 (R#38)
    s.family = F_FOURROOMS;
    s.size = 17;
    s.height = s.width = 17;
    s.max_steps = 100;
    s.n_actions = 7;
  } else if (square("GoToDoor-", F_GOTODOOR)) {
    // [MG] GoToDoorEnv(size): a random room of 5..size cells per side, 4 doors
    if (s.size < 5 || s.size > 16) return false;
    s.max_steps = 4 * s.size * s.size;
    s.n_actions = 7;
  } else if (square("Empty-", F_EMPTY)) {
    if (s.size < 3 || s.size > 16) return false;
    s.max_steps = 4 * s.size * s.size;  // [MG] EmptyEnv
    s.n_actions = 7;
  } else if (square("DoorKey-", F_DOORKEY) || square("DoorKey-Random-", F_DOORKEY)) {
    // DoorKey-Random-SxS: [MG]'s DoorKey already draws the agent's cell and
    // direction, so the Random ids are the same generator (R#36)
    if (s.size < 5 || s.size > 16) return false;
    s.max_steps = 10 * s.size * s.size;  // [MG] DoorKeyEnv
    s.n_actions = 7;
  } else if (square("Dynamic-Obstacles-", F_DYNOBS) ||
             (square("Dynamic-Obstacles-Random-", F_DYNOBS) && (s.random_start = true))) {
    if (s.size < 4 || s.size > 16) return false;
    s.max_steps = 4 * s.size * s.size;  // [MG] DynamicObstaclesEnv
    s.n_actions = 3;                    // Discrete(forward + 1) (R#7)
    // [MG] registrations: 5x5 -> 2, 6x6 -> 3, 8x8 -> 4 (default), 16x16 -> 8;
    // capped to int(size/2) if n > size/2 + 1.
    int n = s.size == 5 ? 2 : s.size == 6 ? 3 : s.size == 16 ? 8 : 4;
    if (!(n <= s.size / 2.0 + 1)) n = s.size / 2;
    s.n_obstacles = n;
  } else if (starts_with(id, "LavaGapS") || starts_with(id, "LavaGap-S")) {
    // Table 8 spells it LavaGapS7, Table 9 LavaGap-S7
    pos = starts_with(id, "LavaGapS") ? 8 : 9;
    int S;
    if (!parse_int(id, pos, &S) || pos != id.size()) return false;
    if (S < 5 || S > 16) return false;
    s.family = F_LAVAGAP;
    s.size = S;
    s.height = s.width = S;
    s.max_steps = 4 * S * S;  // [MG] LavaGapEnv
    s.n_actions = 7;
  } else if (starts_with(id, "KeyCorridorS")) {
    pos = 12;
    int rs, nr;
    if (!parse_int(id, pos, &rs)) return false;
    if (pos >= id.size() || id[pos] != 'R') return false;
    ++pos;
    if (!parse_int(id, pos, &nr) || pos != id.size()) return false;
    if (rs < 3 || nr < 1 || nr > 3) return false;
    s.family = F_KEYCORRIDOR;
    s.room_size = rs;
    s.num_rows = nr;
    s.height = (rs - 1) * nr + 1;  // [MG] RoomGrid
    s.width = (rs - 1) * 3 + 1;
    if (s.width > 16 || s.height > 16) return false;
    s.max_steps = 30 * rs * rs;  // [MG] KeyCorridorEnv
    s.n_actions = 7;
  } else {
    return false;
  }
  *out = s;
  return true;
}

// ---------------------------------------------------------------- reward
// Eq. (1) P:216 read per R#1: success-gated, 1 - 0.9 * (step_count / max_steps)
// with the post-increment step_count, evaluated in binary64 in [MG]'s
// operation order and rounded once to binary32 (R#2).  Compiled with
// -ffp-contract=off so no FMA contraction happens.
float success_reward(int mode, int sc, int T) {
  if (mode == RM_NAVIX) return 1.0f;  // P:223 Markovian reward
  double q = (double)sc / (double)T;
  double p = 0.9 * q;
  double r = 1.0 - p;
  return (float)r;
}

// ---------------------------------------------------------------- step
std::pair<int, int> Env::front_pos() const {
  // [MG] DIR_TO_VEC: 0 (1,0) east, 1 (0,1) south, 2 (-1,0) west, 3 (0,-1) north
  static const int DX[4] = {1, 0, -1, 0};
  static const int DY[4] = {0, 1, 0, -1};
  return {agent_x + DX[agent_dir], agent_y + DY[agent_dir]};
}

StepOut Env::step(int action) {
  StepOut out;
  if (prev_done) {
    // Next-step autoreset ("autoresets when done"; R#18):
    // the action is ignored, episode e+1 starts, reward 0 and flags 0.
    episode += 1;
    generate();
    return out;
  }
  const Spec& S = spec;
  bool not_clear = false;
  if (S.family == F_DYNOBS) {
    // [MG] DynamicObstaclesEnv.step: invalid action -> 0 (R#7)
    if (action >= S.n_actions) action = 0;
    auto fp = front_pos();
    const Cell& front_cell = grid.get(fp.first, fp.second);
    not_clear = front_cell.has_value() && front_cell->type != T_GOAL;  // before the balls move
    // Transition system mu: each ball, in creation order, moves to a
    // uniform admissible cell of its 3x3 box (R#5).  Draw i = word i of the
    // block with counter (env, episode, (1<<16) | step_count, 0).
    DrawStream ds(seed, global_index, episode, (1u << 16) | (uint32_t)step_count);
    for (size_t b = 0; b < obstacles.size(); ++b) {
      uint32_t u = ds.next();
      int ox = obstacles[b].first, oy = obstacles[b].second;
      int tx = std::max(ox - 1, 0), ty = std::max(oy - 1, 0);
      int ex = std::min(tx + 3, grid.width), ey = std::min(ty + 3, grid.height);
      std::vector<std::pair<int, int>> cand;
      for (int y = ty; y < ey; ++y)
        for (int x = tx; x < ex; ++x) {
          if (grid.get(x, y).has_value()) continue;     // [MG] place_obj: not on another object
          if (x == agent_x && y == agent_y) continue;  // [MG] place_obj: not on the agent
          cand.push_back({x, y});
        }
      if (cand.empty()) continue;  // [MG] RecursionError swallowed: the ball stays
      auto c = cand[bounded(u, (uint32_t)cand.size())];
      Cell ball = grid.get(ox, oy);
      grid.set(c.first, c.second, ball);
      grid.set(ox, oy, Cell());
      obstacles[b] = c;
    }
  }

  // [MG] MiniGridEnv.step
  step_count += 1;
  float reward = 0.f;
  bool terminated = false;
  bool success = false, lava = false, collision = false;
  auto fp = front_pos();
  // re-read after the balls moved; outside the grid reads as a Wall, as
  // gen_obs_grid's slice does (R#37: only GoToDoor's open grid edge gets there)
  const bool fp_in = fp.first >= 0 && fp.second >= 0 && fp.first < grid.width && fp.second < grid.height;
  Cell fwd_cell = fp_in ? grid.get(fp.first, fp.second) : Cell(make_wall());
  switch (action) {
    case A_LEFT:
      agent_dir -= 1;
      if (agent_dir < 0) agent_dir += 4;
      break;
    case A_RIGHT:
      agent_dir = (agent_dir + 1) % 4;
      break;
    case A_FORWARD:
      if (!fwd_cell || fwd_cell->can_overlap()) { agent_x = fp.first; agent_y = fp.second; }
      if (fwd_cell && fwd_cell->type == T_GOAL) {
        terminated = true;
        success = true;
        reward = success_reward(reward_mode, step_count, S.max_steps);
      }
      if (fwd_cell && fwd_cell->type == T_LAVA) {
        terminated = true;
        lava = true;
        reward = reward_mode == RM_NAVIX ? -1.0f : 0.0f;  // Table 6 P:572 vs [MG] (R#3)
      }
      break;
    case A_PICKUP:
      if (fwd_cell && fwd_cell->can_pickup()) {
        if (!carrying) {
          carrying = fwd_cell;
          grid.set(fp.first, fp.second, Cell());
        }
      }
      break;
    case A_DROP:
      if (!fwd_cell && carrying) {
        grid.set(fp.first, fp.second, carrying);
        carrying.reset();
      }
      break;
    case A_TOGGLE:
      if (fwd_cell) {
        Obj o = *fwd_cell;
        if (o.type == T_DOOR) {
          // [MG] Door.toggle
          if (o.is_locked) {
            if (carrying && carrying->type == T_KEY && carrying->color == o.color) {
              o.is_locked = false;
              o.is_open = true;
            }
          } else {
            o.is_open = !o.is_open;
          }
          grid.set(fp.first, fp.second, o);
        } else if (o.type == T_BOX) {
          // [MG] Box.toggle: replaced by its contents (always None here)
          grid.set(fp.first, fp.second, Cell());
        }
      }
      break;
    default:
      // done (6) is a no-op; actions >= 7 are no-ops too (R#15)
      break;
  }
  bool failure = false;
  if (S.family == F_GOTODOOR && reward_mode == RM_NAVIX) {
    // Table 6 / Table 7 `on_door_done`: +1 and termination when
    // done is performed in front of the mission's door; nothing else ends the
    // episode (R#39)
    if (action == A_DONE && fp.first == target_x && fp.second == target_y) {
      reward = success_reward(reward_mode, step_count, S.max_steps);
      success = true;
      terminated = true;
    }
  } else if (S.family == F_GOTODOOR) {
    // [MG] GoToDoorEnv.step: toggle ends the episode (the door is already
    // toggled); done ends it, with the success reward iff the agent is next
    // to the target door (R#37)
    if (action == A_TOGGLE) terminated = true;
    if (action == A_DONE) {
      if ((agent_x == target_x && std::abs(agent_y - target_y) == 1) ||
          (agent_y == target_y && std::abs(agent_x - target_x) == 1)) {
        reward = success_reward(reward_mode, step_count, S.max_steps);
        success = true;
      }
      terminated = true;
    }
    failure = (action == A_TOGGLE || action == A_DONE) && !success;  // not lava / goal (imported states)
  }
  if (S.family == F_KEYCORRIDOR && action == A_PICKUP && carrying && carrying->type == T_BALL) {
    // [MG] KeyCorridorEnv.step: picking up the target ball (R#8)
    reward = success_reward(reward_mode, step_count, S.max_steps);
    terminated = true;
    success = true;
  }
  if (S.family == F_DYNOBS && action == A_FORWARD && not_clear) {
    // [MG] DynamicObstaclesEnv.step; R_3 "hit by a flying object" P:973 (R#4)
    reward = -1.0f;
    terminated = true;
    collision = true;
    success = false;
  }
  // Table 6 / Table 7 function selection (R#42): the events are exclusive;
  // a deselected reward function pays 0, a deselected termination function
  // does not end the episode (and the event is not counted in the statistics)
  {
    const bool fail_ev = collision || failure;
    const uint32_t ev = success ? 1u : fail_ev ? 4u : lava ? 2u : 0u;  // [MG]: the collision override wins
    if (ev && !(reward_events & ev)) reward = 0.f;
    if (ev && !(termination_events & ev)) {
      terminated = false;
      success = lava = collision = failure = false;
    }
  }
  bool truncated = (step_count >= S.max_steps) && !terminated;  // R#17
  // Code 4 `compose` of the event reward with time_cost (every step) and
  // action_cost (every action but done), summed in binary32 in this order (R#31)
  if (time_cost != 0.f || action_cost != 0.f) {
    volatile float r = reward;
    r = r + (-time_cost);
    r = r + (action != A_DONE ? -action_cost : 0.f);
    reward = r;
  }
  out.reward = reward;
  out.terminated = terminated;
  out.truncated = truncated;
  prev_done = terminated || truncated;
  if (prev_done) {
    // Episode statistics on the terminal step (info i_{t+1}).
    stats[ST_EPISODES] += 1;
    stats[ST_SUM_LEN] += step_count;
    if (success) { stats[ST_SUCCESS] += 1; stats[ST_SUM_SUCCESS_STEP] += step_count; }
    if (lava) stats[ST_LAVA] += 1;
    if (collision || failure) stats[ST_FAILURE] += 1;
    if (truncated) stats[ST_TRUNCATED] += 1;
  }
  return out;
}

// [MG] MiniGridEnv.gen_obs_grid + Grid.encode(vis_mask): the
// symbolic_first_person observation of Table 5, uint8 (R#10),
// [vi][vj][c] order (R#11), view size 7 (R#14).
void Env::gen_obs(uint8_t* out) const {
  const int R = 7;
  int topX, topY;
  // [MG] get_view_exts
  if (agent_dir == 0) { topX = agent_x; topY = agent_y - R / 2; }
  else if (agent_dir == 1) { topX = agent_x - R / 2; topY = agent_y; }
  else if (agent_dir == 2) { topX = agent_x - R + 1; topY = agent_y - R / 2; }
  else { topX = agent_x - R / 2; topY = agent_y - R + 1; }
  Grid g = grid.slice(topX, topY, R, R);
  for (int i = 0; i < agent_dir + 1; ++i) g = g.rotate_left();
  std::vector<uint8_t> vis = g.process_vis(R / 2, R - 1);
  // the agent sees what it carries (R#13)
  g.set(R / 2, R - 1, carrying);
  g.encode(vis, out);
}

// Table 5 `symbolic`: [MG] FullyObsWrapper — grid.encode() over the
// whole grid (every cell visible) with the agent cell overwritten by
// (OBJECT_TO_IDX["agent"], COLOR_TO_IDX["red"], agent_dir); memory order
// [x][y][c] as Grid.encode returns it (R#32).
void Env::gen_full_obs(uint8_t* out) const {
  std::vector<uint8_t> all((size_t)grid.width * grid.height, 1);
  grid.encode(all, out);
  uint8_t* a = out + ((size_t)agent_x * grid.height + agent_y) * 3;
  a[0] = T_AGENT;
  a[1] = C_RED;
  a[2] = (uint8_t)agent_dir;
}

// ---------------------------------------------------------------- export
int export_bytes_per_env(const Spec& s) {
  return 3 * s.height * s.width + 12 + (s.family == F_DYNOBS ? 2 * s.n_obstacles : 0) +
         (s.family == F_GOTODOOR ? 2 : 0);
}

static void put16(uint8_t* p, uint32_t v) { p[0] = v & 0xff; p[1] = (v >> 8) & 0xff; }
static void put32(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; ++i) p[i] = (v >> (8 * i)) & 0xff; }
static uint32_t get16(const uint8_t* p) { return p[0] | (p[1] << 8); }
static uint32_t get32(const uint8_t* p) { return p[0] | (p[1] << 8) | (p[2] << 16) | ((uint32_t)p[3] << 24); }

// Canonical per-env record: cells (type, colour, state)
// row-major y outer / x inner; agent x, y, dir; carry (type, colour) with
// (1, 0) for nothing; step_count u16; episode u32; prev_done u8; DynObs balls.
void export_env(const Env& e, uint8_t* out) {
  const Spec& s = e.spec;
  uint8_t* p = out;
  for (int y = 0; y < s.height; ++y)
    for (int x = 0; x < s.width; ++x) {
      const Cell& c = e.grid.get(x, y);
      if (c) c->encode(p);
      else { p[0] = T_EMPTY; p[1] = 0; p[2] = 0; }
      p += 3;
    }
  p[0] = (uint8_t)e.agent_x; p[1] = (uint8_t)e.agent_y; p[2] = (uint8_t)e.agent_dir;
  p += 3;
  if (e.carrying) { p[0] = e.carrying->type; p[1] = e.carrying->color; }
  else { p[0] = T_EMPTY; p[1] = 0; }
  p += 2;
  put16(p, (uint32_t)e.step_count); p += 2;
  put32(p, e.episode); p += 4;
  p[0] = e.prev_done ? 1 : 0; p += 1;
  if (s.family == F_DYNOBS)
    for (int b = 0; b < s.n_obstacles; ++b) {
      p[0] = (uint8_t)e.obstacles[b].first; p[1] = (uint8_t)e.obstacles[b].second; p += 2;
    }
  if (s.family == F_GOTODOOR) { p[0] = (uint8_t)e.target_x; p[1] = (uint8_t)e.target_y; }
}

static bool decode_obj(const uint8_t* t, Cell* out) {
  uint8_t type = t[0], color = t[1], state = t[2];
  if (color > 5 || state > 2) return false;
  if (type == T_EMPTY) { if (color || state) return false; out->reset(); return true; }
  Obj o;
  o.type = type;
  o.color = color;
  switch (type) {
    case T_WALL: case T_FLOOR: case T_KEY: case T_BALL: case T_BOX: case T_GOAL: case T_LAVA:
      if (state) return false;
      break;
    case T_DOOR:
      o.is_open = state == 0;
      o.is_locked = state == 2;
      break;
    default:
      return false;
  }
  *out = o;
  return true;
}

bool import_env(Env& e, const uint8_t* in) {
  const Spec& s = e.spec;
  Grid g(s.width, s.height);
  const uint8_t* p = in;
  for (int y = 0; y < s.height; ++y)
    for (int x = 0; x < s.width; ++x) {
      Cell c;
      if (!decode_obj(p, &c)) return false;
      g.set(x, y, c);
      p += 3;
    }
  // closed border of walls (the invariant R#12 relies on); GoToDoor reads
  // outside the grid as walls everywhere (R#37), so its border is free
  const bool open_edge = s.family == F_GOTODOOR;
  for (int y = 0; y < s.height && !open_edge; ++y)
    for (int x = 0; x < s.width; ++x)
      if (x == 0 || y == 0 || x == s.width - 1 || y == s.height - 1) {
        const Cell& c = g.get(x, y);
        if (!c || c->type != T_WALL) return false;
      }
  int ax = p[0], ay = p[1], ad = p[2];
  p += 3;
  const int m = open_edge ? 0 : 1;
  if (ax < m || ay < m || ax > s.width - 1 - m || ay > s.height - 1 - m || ad > 3) return false;
  const Cell& under = g.get(ax, ay);
  if (under && !under->can_overlap()) return false;
  Cell carry;
  uint8_t ct[3] = {p[0], p[1], 0};
  if (!decode_obj(ct, &carry)) return false;
  if (carry && !carry->can_pickup()) return false;
  p += 2;
  int sc = (int)get16(p); p += 2;
  uint32_t ep = get32(p); p += 4;
  int pd = p[0]; p += 1;
  if (pd > 1 || sc > s.max_steps) return false;
  std::vector<std::pair<int, int>> obst;
  if (s.family == F_DYNOBS) {
    for (int b = 0; b < s.n_obstacles; ++b) {
      int bx = p[0], by = p[1];
      p += 2;
      if (bx < 1 || by < 1 || bx > s.width - 2 || by > s.height - 2) return false;
      const Cell& c = g.get(bx, by);
      if (!c || c->type != T_BALL) return false;
      for (auto& q : obst) if (q.first == bx && q.second == by) return false;
      obst.push_back({bx, by});
    }
  }
  int tx = 0, ty = 0;
  if (s.family == F_GOTODOOR) {
    tx = p[0]; ty = p[1];
    if (tx >= s.width || ty >= s.height) return false;
  }
  e.grid = g;
  e.target_x = tx; e.target_y = ty;
  e.agent_x = ax; e.agent_y = ay; e.agent_dir = ad;
  e.carrying = carry;
  e.step_count = sc;
  e.episode = ep;
  e.prev_done = pd != 0;
  e.obstacles = obst;
  return true;
}

}  // namespace oracle
