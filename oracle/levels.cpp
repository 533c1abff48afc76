// oracle/levels.cpp — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
//
// Philox4x32-10 and the level generators (the starting distribution P0 of
// `reset(key)`; Table 9), transcribed from upstream
// MiniGrid's _gen_grid methods (P:206 parity claim; S:446 worlds.generate).
// MiniGrid's rejection loops (`place_obj`, `place_agent`) are replaced by a
// direct uniform draw over the admissible set enumerated row-major (y outer,
// x inner; for (pos, dir) pairs dir innermost): same law, one draw (R#22).
// `connect_all` keeps upstream's loop because its law depends on it.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <functional>

#include "oracle.hpp"

namespace oracle {

// ---------------------------------------------------------------- Philox
// Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as 1, 2, 3",
// SC'11: Philox4x32 with multipliers M0=0xD2511F53, M1=0xCD9E8D57 and Weyl
// key increments W0=0x9E3779B9, W1=0xBB67AE85; 10 rounds, the key bumped
// between rounds.  Pinned by the Random123 known-answer vectors (tests).
void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
    uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
    uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
    uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
    uint32_t y0 = hi1 ^ x1 ^ k0;
    uint32_t y1 = lo1;
    uint32_t y2 = hi0 ^ x3 ^ k1;
    uint32_t y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

uint32_t bounded(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * (uint64_t)n) >> 32); }

DrawStream::DrawStream(uint64_t seed, uint32_t c0_, uint32_t c1_, uint32_t c2_)
    : c0(c0_), c1(c1_), c2(c2_) {
  key[0] = (uint32_t)(seed & 0xffffffffu);
  key[1] = (uint32_t)(seed >> 32);
}
uint32_t DrawStream::next() {
  uint32_t ctr[4] = {c0, c1, c2, (uint32_t)(k / 4)};
  uint32_t out[4];
  philox4x32_10(ctr, key, out);  // recomputed per draw: slow and obviously right
  uint32_t w = out[k % 4];
  k += 1;
  return w;
}

// ---------------------------------------------------------------- helpers
// Uniform over the admissible cells of [top, top+size) clipped to the grid:
// empty (None) cells, not the agent cell, not rejected by `reject`.
// Mirrors [MG] MiniGridEnv.place_obj's acceptance test.
static bool place_uniform(const Env& e, int topx, int topy, int sx, int sy, uint32_t u,
                          const std::function<bool(int, int)>& reject, int* ox, int* oy) {
  topx = std::max(topx, 0);
  topy = std::max(topy, 0);
  int ex = std::min(topx + sx, e.grid.width), ey = std::min(topy + sy, e.grid.height);
  std::vector<std::pair<int, int>> cand;
  for (int y = topy; y < ey; ++y)
    for (int x = topx; x < ex; ++x) {
      if (e.grid.get(x, y).has_value()) continue;
      if (x == e.agent_x && y == e.agent_y) continue;
      if (reject && reject(x, y)) continue;
      cand.push_back({x, y});
    }
  if (cand.empty()) return false;
  auto c = cand[bounded(u, (uint32_t)cand.size())];
  *ox = c.first;
  *oy = c.second;
  return true;
}

// ---------------------------------------------------------------- Empty
// [MG] EmptyEnv._gen_grid: walls, goal at (w-2, h-2), agent (1,1) facing east.
static void gen_empty(Env& e) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.grid.set(W - 2, H - 2, make_goal());
  e.agent_x = 1; e.agent_y = 1; e.agent_dir = 0;
}

// [MG] EmptyEnv._gen_grid with agent_start_pos=None: place_agent() over the
// whole grid (empty cells, the goal excluded), then a random direction.
static void gen_empty_random(Env& e, DrawStream& ds) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.grid.set(W - 2, H - 2, make_goal());
  e.agent_x = -1; e.agent_y = -1;
  int ax, ay;
  place_uniform(e, 0, 0, W, H, ds.next(), nullptr, &ax, &ay);
  e.agent_x = ax; e.agent_y = ay;
  e.agent_dir = (int)ds.next_bounded(4);
}

// [MG] DistShiftEnv._gen_grid: goal (width-2, 1), two lava strips of width-6
// cells from x = 3 on rows 1 and strip2_row, agent (1,1) east.  No draws.
static void gen_distshift(Env& e) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.grid.set(W - 2, 1, make_goal());
  for (int i = 0; i < W - 6; ++i) {
    e.grid.set(3 + i, 1, make_lava());
    e.grid.set(3 + i, e.spec.strip2_row, make_lava());
  }
  e.agent_x = 1; e.agent_y = 1; e.agent_dir = 0;
}

// ---------------------------------------------------------------- Crossing
// [MG] CrossingEnv._gen_grid with obstacle_type = Wall (SimpleCrossing) or
// Lava (Table 9's Crossings, LavaCrossing; R#35), step by step.  The two
// np_random.shuffle calls follow R#35: the rivers list is shuffled by a
// partial Fisher-Yates over its first num_crossings slots (slot k swaps with
// k + bounded(draw, M - k)), which is all [MG] keeps of it; the path is
// shuffled by numpy's Fisher-Yates (for i = n-1 .. 1: swap i with
// bounded(draw, i + 1)).  np_random.choice(range(a, b)) = a + bounded(draw, b - a).
static void gen_crossing(Env& e, DrawStream& ds) {
  const int W = e.spec.width, H = e.spec.height, N = e.spec.n_crossings;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.agent_x = 1; e.agent_y = 1; e.agent_dir = 0;
  e.grid.set(W - 2, H - 2, make_goal());
  // rivers = [(v, i) for i in range(2, H-2, 2)] + [(h, j) for j in range(2, W-2, 2)]
  std::vector<std::pair<char, int>> rivers;
  for (int i = 2; i < H - 2; i += 2) rivers.push_back({'v', i});
  for (int j = 2; j < W - 2; j += 2) rivers.push_back({'h', j});
  const int M = (int)rivers.size();
  for (int k = 0; k < N; ++k) {
    int j = k + (int)ds.next_bounded((uint32_t)(M - k));
    std::swap(rivers[k], rivers[j]);
  }
  rivers.resize(N);
  std::vector<int> rivers_v, rivers_h;
  for (auto& r : rivers) (r.first == 'v' ? rivers_v : rivers_h).push_back(r.second);
  std::sort(rivers_v.begin(), rivers_v.end());
  std::sort(rivers_h.begin(), rivers_h.end());
  // obstacle_pos = product(range(1, W-1), rivers_h) ++ product(rivers_v, range(1, H-1))
  const Obj obstacle = e.spec.lava_obstacle ? make_lava() : make_wall();
  for (int i = 1; i < W - 1; ++i)
    for (int j : rivers_h) e.grid.set(i, j, obstacle);
  for (int i : rivers_v)
    for (int j = 1; j < H - 1; ++j) e.grid.set(i, j, obstacle);
  // path = [h] * len(rivers_v) + [v] * len(rivers_h), shuffled
  std::vector<char> path;
  for (size_t k = 0; k < rivers_v.size(); ++k) path.push_back('h');
  for (size_t k = 0; k < rivers_h.size(); ++k) path.push_back('v');
  for (int i = (int)path.size() - 1; i >= 1; --i) {
    int j = (int)ds.next_bounded((uint32_t)(i + 1));
    std::swap(path[i], path[j]);
  }
  // openings
  std::vector<int> limits_v{0}, limits_h{0};
  for (int v : rivers_v) limits_v.push_back(v);
  limits_v.push_back(H - 1);
  for (int h : rivers_h) limits_h.push_back(h);
  limits_h.push_back(W - 1);
  int room_i = 0, room_j = 0;
  for (char d : path) {
    int i, j;
    if (d == 'h') {
      i = limits_v[room_i + 1];
      j = limits_h[room_j] + 1 + (int)ds.next_bounded((uint32_t)(limits_h[room_j + 1] - limits_h[room_j] - 1));
      room_i += 1;
    } else {
      i = limits_v[room_i] + 1 + (int)ds.next_bounded((uint32_t)(limits_v[room_i + 1] - limits_v[room_i] - 1));
      j = limits_h[room_j + 1];
      room_j += 1;
    }
    e.grid.set(i, j, std::nullopt);
  }
}

// ---------------------------------------------------------------- FourRooms
// [MG] FourRoomsEnv._gen_grid, step by step: outer walls; for each room
// (j outer, i inner) its right wall with one opening, then its bottom wall
// with one opening; place_agent() over the whole grid, then place_obj(Goal).
static void gen_fourrooms(Env& e, DrawStream& ds) {
  const int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.horz_wall(0, 0, -1, make_wall());
  e.grid.horz_wall(0, H - 1, -1, make_wall());
  e.grid.vert_wall(0, 0, -1, make_wall());
  e.grid.vert_wall(W - 1, 0, -1, make_wall());
  const int room_w = W / 2, room_h = H / 2;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) {
      const int xL = i * room_w, yT = j * room_h, xR = xL + room_w, yB = yT + room_h;
      if (i + 1 < 2) {
        e.grid.vert_wall(xR, yT, room_h, make_wall());
        const int y = yT + 1 + (int)ds.next_bounded((uint32_t)(yB - yT - 1));  // _rand_int(yT + 1, yB)
        e.grid.set(xR, y, Cell());
      }
      if (j + 1 < 2) {
        e.grid.horz_wall(xL, yB, room_w, make_wall());
        const int x = xL + 1 + (int)ds.next_bounded((uint32_t)(xR - xL - 1));  // _rand_int(xL + 1, xR)
        e.grid.set(x, yB, Cell());
      }
    }
  e.agent_x = -1; e.agent_y = -1;
  int ax, ay;
  place_uniform(e, 0, 0, W, H, ds.next(), nullptr, &ax, &ay);
  e.agent_x = ax; e.agent_y = ay;
  e.agent_dir = (int)ds.next_bounded(4);
  int gx, gy;
  place_uniform(e, 0, 0, W, H, ds.next(), nullptr, &gx, &gy);
  e.grid.set(gx, gy, make_goal());
}

// ---------------------------------------------------------------- GoToDoor
// [MG] GoToDoorEnv._gen_grid, step by step.  _rand_int(a, b) = a +
// bounded(draw, b - a); the colour loop (rand_elem until unused) is one draw
// over the unused colours in COLOR_NAMES order (R#37, as R#20).
static void gen_gotodoor(Env& e, DrawStream& ds) {
  const int S = e.spec.size;
  e.grid = Grid(S, S);
  const int w = 5 + (int)ds.next_bounded((uint32_t)(S + 1 - 5));
  const int h = 5 + (int)ds.next_bounded((uint32_t)(S + 1 - 5));
  e.grid.wall_rect(0, 0, w, h);
  int dx[4], dy[4];
  dx[0] = 2 + (int)ds.next_bounded((uint32_t)(w - 4)); dy[0] = 0;
  dx[1] = 2 + (int)ds.next_bounded((uint32_t)(w - 4)); dy[1] = h - 1;
  dx[2] = 0; dy[2] = 2 + (int)ds.next_bounded((uint32_t)(h - 4));
  dx[3] = w - 1; dy[3] = 2 + (int)ds.next_bounded((uint32_t)(h - 4));
  std::vector<int> unused{0, 1, 2, 3, 4, 5}, colors;
  while (colors.size() < 4) {
    int k = (int)ds.next_bounded((uint32_t)unused.size());
    colors.push_back(unused[k]);
    unused.erase(unused.begin() + k);
  }
  for (int i = 0; i < 4; ++i) e.grid.set(dx[i], dy[i], make_door((uint8_t)colors[i], false));
  // place_agent(size=(w, h)): position then direction
  e.agent_x = -1; e.agent_y = -1;
  int ax, ay;
  place_uniform(e, 0, 0, w, h, ds.next(), nullptr, &ax, &ay);
  e.agent_x = ax; e.agent_y = ay;
  e.agent_dir = (int)ds.next_bounded(4);
  const int t = (int)ds.next_bounded(4);
  e.target_x = dx[t]; e.target_y = dy[t];
}

// ---------------------------------------------------------------- DoorKey
// [MG] DoorKeyEnv._gen_grid (SURVEY §8c-4 draw order d0..d4).
static void gen_doorkey(Env& e, DrawStream& ds) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.grid.set(W - 2, H - 2, make_goal());
  int split = 2 + (int)ds.next_bounded((uint32_t)(W - 4));  // _rand_int(2, width-2)
  e.grid.vert_wall(split, 0, -1, make_wall());
  // place_agent(size=(splitIdx, height)): position then direction
  e.agent_x = -1; e.agent_y = -1;
  int ax, ay;
  place_uniform(e, 0, 0, split, H, ds.next(), nullptr, &ax, &ay);
  e.agent_x = ax; e.agent_y = ay;
  e.agent_dir = (int)ds.next_bounded(4);
  int door_y = 1 + (int)ds.next_bounded((uint32_t)(W - 3));  // _rand_int(1, width-2) (R#24)
  e.grid.set(split, door_y, make_door(C_YELLOW, true));
  int kx, ky;
  place_uniform(e, 0, 0, split, H, ds.next(), nullptr, &kx, &ky);
  e.grid.set(kx, ky, make_key(C_YELLOW));
}

// ---------------------------------------------------------------- LavaGap
// [MG] LavaGapEnv._gen_grid.
static void gen_lavagap(Env& e, DrawStream& ds) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.agent_x = 1; e.agent_y = 1; e.agent_dir = 0;
  e.grid.set(W - 2, H - 2, make_goal());
  int gx = 2 + (int)ds.next_bounded((uint32_t)(W - 4));  // _rand_int(2, width-2)
  int gy = 1 + (int)ds.next_bounded((uint32_t)(H - 2));  // _rand_int(1, height-1)
  e.grid.vert_wall(gx, 1, H - 2, make_lava());
  e.grid.set(gx, gy, Cell());
}

// ---------------------------------------------------------------- DynObs
// [MG] DynamicObstaclesEnv._gen_grid: Empty layout, agent (1,1) east, then
// n blue balls, each uniform over the empty cells except the agent's.
static void gen_dynobs(Env& e, DrawStream& ds) {
  int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  e.grid.wall_rect(0, 0, W, H);
  e.grid.set(W - 2, H - 2, make_goal());
  if (e.spec.random_start) {
    // [MG] DynamicObstaclesEnv(agent_start_pos=None): place_agent(), then the balls
    e.agent_x = -1; e.agent_y = -1;
    int ax, ay;
    place_uniform(e, 0, 0, W, H, ds.next(), nullptr, &ax, &ay);
    e.agent_x = ax; e.agent_y = ay;
    e.agent_dir = (int)ds.next_bounded(4);
  } else {
    e.agent_x = 1; e.agent_y = 1; e.agent_dir = 0;
  }
  e.obstacles.clear();
  for (int i = 0; i < e.spec.n_obstacles; ++i) {
    int bx, by;
    if (!place_uniform(e, 0, 0, W, H, ds.next(), nullptr, &bx, &by)) {
      e.stats[ST_GEN_FAIL] += 1;
      continue;
    }
    e.grid.set(bx, by, make_ball(C_BLUE));
    e.obstacles.push_back({bx, by});
  }
}

// ---------------------------------------------------------------- KeyCorridor
// [MG] RoomGrid._gen_grid + KeyCorridorEnv._gen_grid + RoomGrid.connect_all.
namespace {
struct Room {
  int top_x, top_y, size_x, size_y;
  bool has_door_pos[4] = {false, false, false, false};
  int door_pos[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  int neighbor[4] = {-1, -1, -1, -1};  // room index j*num_cols+i, or -1
  bool link[4] = {false, false, false, false};  // room.doors[k] is truthy
  bool locked = false;
};
}  // namespace

static void gen_keycorridor(Env& e, DrawStream& ds) {
  const int s = e.spec.room_size, nr = e.spec.num_rows, nc = 3;
  const int W = e.spec.width, H = e.spec.height;
  e.grid = Grid(W, H);
  std::vector<Room> rooms(nr * nc);
  auto room = [&](int i, int j) -> Room& { return rooms[j * nc + i]; };
  for (int j = 0; j < nr; ++j)
    for (int i = 0; i < nc; ++i) {
      Room& r = room(i, j);
      r.top_x = i * (s - 1);
      r.top_y = j * (s - 1);
      r.size_x = s;
      r.size_y = s;
      e.grid.wall_rect(r.top_x, r.top_y, s, s);
    }
  for (int j = 0; j < nr; ++j)
    for (int i = 0; i < nc; ++i) {
      Room& r = room(i, j);
      int x_l = r.top_x + 1, y_l = r.top_y + 1;
      int x_m = r.top_x + r.size_x - 1, y_m = r.top_y + r.size_y - 1;
      if (i < nc - 1) {
        r.neighbor[0] = j * nc + (i + 1);
        r.has_door_pos[0] = true;
        r.door_pos[0][0] = x_m;
        r.door_pos[0][1] = y_l + (int)ds.next_bounded((uint32_t)(y_m - y_l));  // _rand_int(y_l, y_m)
      }
      if (j < nr - 1) {
        r.neighbor[1] = (j + 1) * nc + i;
        r.has_door_pos[1] = true;
        r.door_pos[1][0] = x_l + (int)ds.next_bounded((uint32_t)(x_m - x_l));  // _rand_int(x_l, x_m)
        r.door_pos[1][1] = y_m;
      }
      if (i > 0) {
        r.neighbor[2] = j * nc + (i - 1);
        Room& nb = room(i - 1, j);
        r.has_door_pos[2] = nb.has_door_pos[0];
        r.door_pos[2][0] = nb.door_pos[0][0];
        r.door_pos[2][1] = nb.door_pos[0][1];
      }
      if (j > 0) {
        r.neighbor[3] = (j - 1) * nc + i;
        Room& nb = room(i, j - 1);
        r.has_door_pos[3] = nb.has_door_pos[1];
        r.door_pos[3][0] = nb.door_pos[1][0];
        r.door_pos[3][1] = nb.door_pos[1][1];
      }
    }
  // default agent position of RoomGrid._gen_grid
  e.agent_x = (nc / 2) * (s - 1) + s / 2;
  e.agent_y = (nr / 2) * (s - 1) + s / 2;
  e.agent_dir = 0;

  auto link_rooms = [&](int i, int j, int k) {
    Room& r = room(i, j);
    r.link[k] = true;
    rooms[r.neighbor[k]].link[(k + 2) % 4] = true;
  };
  // KeyCorridor: connect the middle column rooms into a hallway
  // (remove_wall(1, j, 3) for j = 1..num_rows-1)
  for (int j = 1; j < nr; ++j) {
    Room& r = room(1, j);
    for (int t = 1; t < r.size_x - 1; ++t) e.grid.set(r.top_x + t, r.top_y, Cell());
    link_rooms(1, j, 3);
  }
  // locked door on the left wall of room (2, room_idx), random colour
  int room_idx = (int)ds.next_bounded((uint32_t)nr);
  uint8_t door_color = (uint8_t)ds.next_bounded(6);  // _rand_color (R#23)
  {
    Room& r = room(2, room_idx);
    r.locked = true;
    e.grid.set(r.door_pos[2][0], r.door_pos[2][1], make_door(door_color, true));
    link_rooms(2, room_idx, 2);
  }
  // [MG] reject_next_to: Manhattan distance to the (default) agent pos < 2 (R#25)
  auto reject_next_to = [&](int x, int y) {
    int d = std::abs(e.agent_x - x) + std::abs(e.agent_y - y);
    return d < 2;
  };
  // the target ball behind the locked door: colour, then position
  {
    uint8_t ball_color = (uint8_t)ds.next_bounded(6);
    Room& r = room(2, room_idx);
    int bx, by;
    if (place_uniform(e, r.top_x, r.top_y, r.size_x, r.size_y, ds.next(), reject_next_to, &bx, &by))
      e.grid.set(bx, by, make_ball(ball_color));
    else
      e.stats[ST_GEN_FAIL] += 1;
  }
  // the key in a random room of the left column, in the door's colour
  {
    int kr = (int)ds.next_bounded((uint32_t)nr);
    Room& r = room(0, kr);
    int kx, ky;
    if (place_uniform(e, r.top_x, r.top_y, r.size_x, r.size_y, ds.next(), reject_next_to, &kx, &ky))
      e.grid.set(kx, ky, make_key(door_color));
    else
      e.stats[ST_GEN_FAIL] += 1;
  }
  // [MG] RoomGrid.place_agent(1, num_rows // 2): (pos, dir) uniform over the
  // pairs whose front cell is None or a wall, pos an empty cell of the room.
  {
    Room& r = room(1, nr / 2);
    static const int DX[4] = {1, 0, -1, 0};
    static const int DY[4] = {0, 1, 0, -1};
    std::vector<std::array<int, 3>> cand;
    for (int y = r.top_y; y < std::min(r.top_y + r.size_y, H); ++y)
      for (int x = r.top_x; x < std::min(r.top_x + r.size_x, W); ++x) {
        if (e.grid.get(x, y).has_value()) continue;
        for (int d = 0; d < 4; ++d) {
          const Cell& f = e.grid.get(x + DX[d], y + DY[d]);
          if (!f || f->type == T_WALL) cand.push_back({x, y, d});
        }
      }
    uint32_t u = ds.next();
    if (cand.empty()) {
      e.stats[ST_GEN_FAIL] += 1;
    } else {
      auto c = cand[bounded(u, (uint32_t)cand.size())];
      e.agent_x = c[0]; e.agent_y = c[1]; e.agent_dir = c[2];
    }
  }
  // [MG] RoomGrid.connect_all(max_itrs=5000)
  {
    int start = (e.agent_y / (s - 1)) * nc + (e.agent_x / (s - 1));  // room_from_pos
    int num_itrs = 0;
    while (true) {
      if (num_itrs > 5000) {  // [MG] raises RecursionError; here: counted
        e.stats[ST_GEN_FAIL] += 1;
        break;
      }
      num_itrs += 1;
      // find_reach: DFS over room links from the start room
      std::vector<bool> reach(rooms.size(), false);
      std::vector<int> stack{start};
      int n_reach = 0;
      while (!stack.empty()) {
        int ri = stack.back();
        stack.pop_back();
        if (reach[ri]) continue;
        reach[ri] = true;
        n_reach += 1;
        for (int k = 0; k < 4; ++k)
          if (rooms[ri].link[k]) stack.push_back(rooms[ri].neighbor[k]);
      }
      if (n_reach == (int)rooms.size()) break;
      int i = (int)ds.next_bounded(nc);
      int j = (int)ds.next_bounded((uint32_t)nr);
      int k = (int)ds.next_bounded(4);
      Room& r = room(i, j);
      if (!r.has_door_pos[k] || r.link[k]) continue;
      Room& nb = rooms[r.neighbor[k]];
      if (r.locked || nb.locked) continue;
      uint8_t color = (uint8_t)ds.next_bounded(6);
      e.grid.set(r.door_pos[k][0], r.door_pos[k][1], make_door(color, false));
      link_rooms(i, j, k);
    }
  }
}

// ---------------------------------------------------------------- dispatch
// Level stream: counter (global env index, episode, domain 0 << 16 | 0, block).
void Env::generate() {
  DrawStream ds(seed, global_index, episode, 0u);
  carrying.reset();
  obstacles.clear();
  switch (spec.family) {
    case F_EMPTY: gen_empty(*this); break;
    case F_DOORKEY: gen_doorkey(*this, ds); break;
    case F_DYNOBS: gen_dynobs(*this, ds); break;
    case F_KEYCORRIDOR: gen_keycorridor(*this, ds); break;
    case F_LAVAGAP: gen_lavagap(*this, ds); break;
    case F_EMPTY_RANDOM: gen_empty_random(*this, ds); break;
    case F_DISTSHIFT: gen_distshift(*this); break;
    case F_CROSSING: gen_crossing(*this, ds); break;
    case F_GOTODOOR: gen_gotodoor(*this, ds); break;
    case F_FOURROOMS: gen_fourrooms(*this, ds); break;
  }
  step_count = 0;
  prev_done = false;
}

}  // namespace oracle
