// levelgen.cuh — device level generators: the starting distribution P0 of
// reset(key) for the Table 9 families, with
// MiniGrid's layouts.  One thread generates one env's level into its
// SMEM row lines.  Draws follow DESIGN.md R#20-R#25: Philox stream
// (global env, episode, 0, block); rejection loops replaced by one uniform
// draw over the admissible set in row-major order; connect_all keeps its loop.
#pragma once
#include <type_traits>
#include "layout.h"
#include "philox.cuh"

namespace navix {

// Compile-time configuration of one kernel instantiation.
template <int FAM, int H, int W>
struct Cfg {
  static constexpr int RW = (W + 7) / 8;             // u64 planes per grid row (f2: 16- / 24-byte rows)
  static constexpr int NPL = RW == 1 ? 8 : RW * H;  // SMEM planes per env (8 lines / H rows x RW)
  static constexpr int RS = (W - 1) / 3 + 1;         // KeyCorridor room size (3 columns of rooms)
  static constexpr int NR = (H - 1) / (RS - 1);      // KeyCorridor rows
  static constexpr int T = FAM == FAM_DOORKEY ? 10 * W * W
                         : FAM == FAM_KEYCORRIDOR ? 30 * RS * RS
                         : FAM == FAM_FOURROOMS ? 100
                         : 4 * W * H;                // R#16
  static constexpr int NA = FAM == FAM_DYNOBS ? 3 : 7;
  static constexpr int NOBST = FAM != FAM_DYNOBS ? 0 : (W == 5 ? 2 : W == 6 ? 3 : W == 16 ? 8 : 4);  // R#6
};

// Families whose every level has the same layout (template_plane below):
// only the agent and, in Dynamic-Obstacles, the see-through balls differ.
template <int FAM>
constexpr bool STATIC_LAYOUT = FAM == FAM_DYNOBS || FAM == FAM_EMPTY || FAM == FAM_EMPTY_RANDOM ||
                               FAM == FAM_DISTSHIFT1 || FAM == FAM_DISTSHIFT2;

// DoorKey (grids <= 8 wide): the only opaque cells of a generated level are
// the border, the wall column at x = split and its door at (split, door_y),
// whose state the agent can toggle; keys, balls, boxes and the goal are
// see-through and nothing can create an opaque cell.  So the visibility is a
// function of (pose, split, door_y, door open) (step_kernel.cuh vis table).
template <int FAM, int W>
constexpr bool LAYOUT_KEYED_VIS = FAM == FAM_DOORKEY && W <= 8;
// LavaGap and the lava Crossings: lava is see-through, so a generated level's
// only opaque cells are the border; with no door in the grid no action can
// create one.  Their visibility is a function of the pose alone.
template <int FAM>
constexpr bool BORDER_OPACITY = FAM == FAM_LAVAGAP || FAM == FAM_CROSSING;

// Static layout plane p (row y = p / RW, cells x = 8 (p % RW) .. +7) as 8
// cell bytes (cells x >= W are 0 = outside the grid).
template <int FAM, int H, int W>
__host__ __device__ constexpr uint64_t template_plane(int p) {
  constexpr int RW = (W + 7) / 8;
  const int y = p / RW, x0 = 8 * (p % RW);
  uint64_t r = 0;
  for (int x = x0; x < x0 + 8 && x < W; ++x) {
    bool wall = false;
    if (FAM == FAM_GOTODOOR) wall = false;  // the generator draws the room
    else if (FAM == FAM_KEYCORRIDOR) wall = (x % (Cfg<FAM, H, W>::RS - 1) == 0) || (y % (Cfg<FAM, H, W>::RS - 1) == 0);
    else wall = x == 0 || y == 0 || x == W - 1 || y == H - 1;
    uint8_t c = wall ? CELL_WALL : CELL_EMPTY;
    if (FAM == FAM_DISTSHIFT1 || FAM == FAM_DISTSHIFT2) {
      // [MG] DistShiftEnv: goal (W-2, 1), lava x = 3 .. W-4 on rows 1 and strip2_row (R#33)
      const int strip2 = FAM == FAM_DISTSHIFT1 ? 2 : 5;
      if (x == W - 2 && y == 1) c = CELL_GOAL;
      if (x >= 3 && x < W - 3 && (y == 1 || y == strip2)) c = CELL_LAVA;
    } else if (FAM == FAM_FOURROOMS) {
      if (x == W / 2 || y == H / 2) c = CELL_WALL;  // the inner walls; the generator opens 4 gaps
    } else if (FAM != FAM_KEYCORRIDOR && FAM != FAM_GOTODOOR && x == W - 2 && y == H - 2) {
      c = CELL_GOAL;  // goal (W-2, H-2)
    }
    r |= (uint64_t)c << (8 * (x - x0));
  }
  return r;
}

// Bitboard (bit 8y + x) of the empty cells of the static layout, grids up to 8 wide.
template <int FAM, int H, int W>
__host__ __device__ constexpr uint64_t template_free_cells() {
  uint64_t m = 0;
  for (int y = 0; y < H && y < 8; ++y) {
    const uint64_t r = template_plane<FAM, H, W>(y);
    for (int x = 0; x < 8; ++x)
      if (((r >> (8 * x)) & 0xFF) == CELL_EMPTY) m |= 1ull << (8 * y + x);
  }
  return m;
}

// Bitboard of the interior cells (not the border), grids up to 8 wide.
template <int H, int W>
__host__ __device__ constexpr uint64_t interior_cells() {
  uint64_t m = 0;
  for (int y = 1; y < H - 1 && y < 8; ++y)
    for (int x = 1; x < W - 1 && x < 8; ++x) m |= 1ull << (8 * y + x);
  return m;
}

// 0xFF in byte i of the result iff bit i of b (b < 256): each half
// replicates its 4 bits to 4 bytes, keeps bit i in byte i, and the byte's
// sign after + 0x7F (no carry out: bytes <= 8) is replicated by a byte permute.
__device__ __forceinline__ uint64_t bits_to_bytes(uint32_t b) {
  uint32_t lo = ((b & 0xFu) * 0x01010101u & 0x08040201u) + 0x7F7F7F7Fu;
  uint32_t hi = ((b >> 4) * 0x01010101u & 0x08040201u) + 0x7F7F7F7Fu;
  asm("prmt.b32 %0, %0, 0, 0xBA98;" : "+r"(lo));
  asm("prmt.b32 %0, %0, 0, 0xBA98;" : "+r"(hi));
  return ((uint64_t)hi << 32) | lo;
}

// Byte mask of the interior cells (1 <= x <= W-2) of row plane q (cells 8q .. 8q+7).
template <int W>
__host__ __device__ constexpr uint64_t interior_bytes(int q) {
  uint64_t m = 0;
  for (int i = 0; i < 8; ++i)
    if (8 * q + i >= 1 && 8 * q + i <= W - 2) m |= 0xFFull << (8 * i);
  return m;
}

// Per-thread view of its env's SMEM rows: plane y * RW + x / 8 holds cells
// x..x+7 of row y (stride TILE between planes).
template <int RW>
struct RowViewT {
  uint64_t* rows;  // &planes[0][tid]
  __device__ __forceinline__ uint8_t* at(int x, int y) const {
    if constexpr (RW == 1)  // one plane per row: x is the byte within it (x < 8)
      return reinterpret_cast<uint8_t*>(rows) + y * (TILE * 8) + x;
    return reinterpret_cast<uint8_t*>(rows + (y * RW + (x >> 3)) * TILE) + (x & 7);
  }
  __device__ __forceinline__ uint8_t get(int x, int y) const { return *at(x, y); }
  __device__ __forceinline__ void set(int x, int y, uint8_t v) const { *at(x, y) = v; }
};

// k-th (0-based) set bit of a 64-bit mask, by binary search on popcounts.
__device__ __forceinline__ int select64(uint64_t m, uint32_t k) {
  int pos = 0;
  uint32_t w = (uint32_t)m;
  uint32_t c = __popc(w);
  if (k >= c) { k -= c; w = (uint32_t)(m >> 32); pos = 32; }
  c = __popc(w & 0xFFFFu);
  if (k >= c) { k -= c; w >>= 16; pos += 16; }
  c = __popc(w & 0xFFu);
  if (k >= c) { k -= c; w >>= 8; pos += 8; }
  c = __popc(w & 0xFu);
  if (k >= c) { k -= c; w >>= 4; pos += 4; }
  c = __popc(w & 0x3u);
  if (k >= c) { k -= c; w >>= 2; pos += 2; }
  c = w & 1u;
  if (k >= c) pos += 1;
  return pos;
}

struct GenOut {
  int ax, ay, dir;
  uint64_t balls;  // DynObs: byte b = ball_code(W, x, y) of ball b (up to 8)
  uint32_t fail;
  uint32_t target;  // GoToDoor: target door (x << 4) | y
};

// bit p of a multi-word mask as word w's part (0 unless p is in word w), in
// arithmetic form: an `if (w == p >> 6)` over unrolled words is turned back
// into an indexed store by the compiler, which moves the mask to local memory.
__device__ __forceinline__ uint64_t word_bit(int p, int w) {
  const unsigned d = (unsigned)(p - 64 * w);
  return (uint64_t)(d < 64u) << (d & 63u);
}

// k-th set bit of a multi-word mask (word w covers bits 64w ..), -1 if fewer.
// The word holding it is picked with selects over the unrolled words (no early
// return, no dynamic index), so the mask stays in registers: an early-exit
// loop put the DynObs-16x16 free-cell mask in local memory (LDL/STL).
template <int NW>
__device__ __forceinline__ int select_bits(const uint64_t (&m)[NW], uint32_t k) {
  uint64_t word = 0;
  int base = -1;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t c = __popcll(m[w]);
    const bool here = base < 0 && k < c;
    word = here ? m[w] : word;
    base = here ? 64 * w : base;
    k = (base < 0) ? k - c : k;
  }
  return base < 0 ? -1 : base + select64(word, k);
}

// word t (0..7) of the two consecutive Philox blocks (x0, x1)
__device__ __forceinline__ uint32_t pick8(const uint4& x0, const uint4& x1, uint32_t t) {
  const uint4& x = t < 4 ? x0 : x1;
  const uint32_t u = t & 3;
  return u == 0 ? x.x : u == 1 ? x.y : u == 2 ? x.z : x.w;
}

// The draws of one level, cached across a warp that generates it together
// (generate_level<..., WARP = true>): lane l holds Philox block base + l of
// the stream (env, episode, 0, block), so 128 consecutive draws cost ONE
// parallel Philox evaluation instead of 32 sequential ones, and any draw is a
// shuffle away.  Same draws as DrawStream, in the same order.
struct WarpDraws {
  uint32_t c0, c1, k0, k1;
  uint32_t base;  // block held by lane 0
  uint32_t pos;   // next draw index (DrawStream::pos)
  uint4 blk;      // this lane's block: base + lane
  __device__ WarpDraws(uint32_t env, uint32_t episode, uint32_t key_lo, uint32_t key_hi)
      : c0(env), c1(episode), k0(key_lo), k1(key_hi), base(0), pos(0) {
    refill(0);
  }
  __device__ __forceinline__ void refill(uint32_t b) {  // warp-uniform b
    base = b;
    blk = philox4x32_10(make_uint4(c0, c1, 0u, b + (threadIdx.x & 31)), k0, k1);
  }
  // block b (cached: b - base < 32, warp-uniform or not) from its lane
  __device__ __forceinline__ uint4 block(uint32_t b) const {
    const int src = (int)(b - base);
    return make_uint4(__shfl_sync(0xffffffffu, blk.x, src), __shfl_sync(0xffffffffu, blk.y, src),
                      __shfl_sync(0xffffffffu, blk.z, src), __shfl_sync(0xffffffffu, blk.w, src));
  }
  // make blocks [b, b + n) resident (warp-uniform b, n <= 32)
  __device__ __forceinline__ void ensure(uint32_t b, uint32_t n) {
    if (b < base || b + n > base + 32u) refill(b);
  }
  __device__ __forceinline__ uint32_t next() {  // warp-uniform
    const uint32_t k = pos++;
    ensure(k >> 2, 1);
    const uint32_t t = k & 3;
    const uint32_t mine = t == 0 ? blk.x : t == 1 ? blk.y : t == 2 ? blk.z : blk.w;
    return __shfl_sync(0xffffffffu, mine, (int)((k >> 2) - base));
  }
  __device__ __forceinline__ uint32_t next_bounded(uint32_t n) { return bounded(next(), n); }
};

// A generator with a fixed draw sequence (no data-dependent branch around a
// draw): its NB Philox blocks are computed up front, independent of each
// other (instruction-level parallelism instead of NB chained evaluations),
// and every draw's block and word are compile-time constants after inlining.
template <int NB>
struct FixedDraws {
  uint4 b[NB];
  uint32_t pos;
  __device__ FixedDraws(uint32_t env, uint32_t episode, uint32_t klo, uint32_t khi) : pos(0) {
#pragma unroll
    for (int i = 0; i < NB; ++i) b[i] = philox4x32_10(make_uint4(env, episode, 0u, (uint32_t)i), klo, khi);
  }
  __device__ __forceinline__ uint32_t next() {
    const uint32_t k = pos++;
    const uint4& x = b[k >> 2];
    const uint32_t t = k & 3;
    return t == 0 ? x.x : t == 1 ? x.y : t == 2 ? x.z : x.w;
  }
  __device__ __forceinline__ uint32_t next_bounded(uint32_t n) { return bounded(next(), n); }
};

// The draw source of generate_level: one thread's DrawStream, the warp's
// cache (KeyCorridor generated by a whole warp), or the prefetched blocks of
// a fixed draw sequence (GoToDoor 13 draws, DoorKey 5, FourRooms 7, LavaGap
// and Empty-Random 2; the Crossings pick theirs per crossing count).
template <int FAM, bool WARP>
struct LevelDrawsT {
  using type = DrawStream;
};
template <bool WARP>
struct LevelDrawsT<FAM_KEYCORRIDOR, WARP> {
  using type = typename std::conditional<WARP, WarpDraws, DrawStream>::type;
};
template <bool WARP>
struct LevelDrawsT<FAM_GOTODOOR, WARP> {
  using type = FixedDraws<4>;
};
template <bool WARP>
struct LevelDrawsT<FAM_DOORKEY, WARP> {
  using type = FixedDraws<2>;
};
template <bool WARP>
struct LevelDrawsT<FAM_FOURROOMS, WARP> {
  using type = FixedDraws<2>;
};
template <bool WARP>
struct LevelDrawsT<FAM_LAVAGAP, WARP> {  // the gap column and row
  using type = FixedDraws<1>;
};
template <bool WARP>
struct LevelDrawsT<FAM_EMPTY_RANDOM, WARP> {  // the agent's cell and direction
  using type = FixedDraws<1>;
};
__device__ __forceinline__ DrawStream make_draws(DrawStream*, uint32_t env, uint32_t ep, uint32_t klo, uint32_t khi) {
  return DrawStream(env, ep, 0u, klo, khi);
}
template <class D>
__device__ __forceinline__ D make_draws(D*, uint32_t env, uint32_t ep, uint32_t klo, uint32_t khi) {
  return D(env, ep, klo, khi);
}

// [MG] CrossingEnv._gen_grid, obstacle Wall or Lava (gparam & CROSSING_LAVA),
// N crossings (NC > 0: N == NC, a compile-time constant, loops unrolled); the
// two shuffles as R#35 reads them.  Rivers are nibbles (bit 3: horizontal,
// bits 0-2: position / 2 - 1): (S-3)/2 vertical ones, then as many horizontal.
template <int H, int W, int NC, class Draws>
__device__ __forceinline__ void crossing_level(RowViewT<Cfg<FAM_CROSSING, H, W>::RW> g, Draws& ds, int N_,
                                               uint8_t obstacle) {
  using C = Cfg<FAM_CROSSING, H, W>;
  constexpr int FAM = FAM_CROSSING;
  constexpr int NRV = (W - 3) / 2, M = 2 * NRV;
  const int N = NC > 0 ? NC : N_;
  constexpr int NU = NC > 0 ? NC : 1;  // unroll factor of the N-long loops
  using RivT = typename std::conditional<(M <= 8), uint32_t, uint64_t>::type;
  RivT riv = 0;
#pragma unroll
  for (int k = 0; k < M; ++k) riv |= (RivT)((k < NRV ? 0 : 8) | (k % NRV)) << (4 * k);
  uint32_t vmask = 0, hmask = 0;  // bit p: a vertical river at x = p / a horizontal one at y = p
#pragma unroll NU
  for (int k = 0; k < N; ++k) {
    const int j = k + (int)ds.next_bounded((uint32_t)(M - k));
    const RivT a = (riv >> (4 * k)) & 15, b = (riv >> (4 * j)) & 15;
    riv = (riv & ~((RivT)15 << (4 * k)) & ~((RivT)15 << (4 * j))) | (b << (4 * k)) | (a << (4 * j));
    const uint32_t bit = 1u << (2 * (((uint32_t)b & 7) + 1));
    if (b & 8) hmask |= bit; else vmask |= bit;
  }
  // the rivers, a whole row plane at a time: plane q of an interior row is
  // obstacle at the interior bytes if the row is a horizontal river, else at
  // the vertical rivers' bytes (a byte mask spread from vmask's bits)
  {
    const uint64_t obst8 = 0x0101010101010101ull * obstacle;
    uint64_t vm[C::RW];
#pragma unroll
    for (int q = 0; q < C::RW; ++q) vm[q] = bits_to_bytes((vmask >> (8 * q)) & 0xFFu);
#pragma unroll
    for (int y = 1; y < H - 1; ++y) {
      const bool hr = (hmask >> y) & 1u;
#pragma unroll
      for (int q = 0; q < C::RW; ++q) {
        const uint64_t m = hr ? interior_bytes<W>(q) : vm[q];
        g.rows[(y * C::RW + q) * TILE] = (template_plane<FAM, H, W>(y * C::RW + q) & ~m) | (obst8 & m);
      }
    }
  }
  // path: popc(vmask) 'h' moves then popc(hmask) 'v' moves (bit k = 1: 'v'), Fisher-Yates
  const int nv = __popc(vmask);
  uint32_t path = ((1u << N) - 1) & ~((1u << nv) - 1);
#pragma unroll NU
  for (int t = 0; t < N - 1; ++t) {
    const int i = N - 1 - t;
    const int j = (int)ds.next_bounded((uint32_t)(i + 1));
    const uint32_t bi = (path >> i) & 1u, bj = (path >> j) & 1u;
    path = (path & ~(1u << i) & ~(1u << j)) | (bj << i) | (bi << j);
  }
  // openings: the current room spans x in (xlo, xhi), y in (ylo, yhi)
  auto next_limit = [](uint32_t m, int lo, int end) {
    const uint32_t above = m & ~((2u << lo) - 1);
    return above ? __ffs(above) - 1 : end;
  };
  int xlo = 0, ylo = 0;
  int xhi = next_limit(vmask, 0, W - 1), yhi = next_limit(hmask, 0, H - 1);
#pragma unroll NU
  for (int k = 0; k < N; ++k) {
    if (((path >> k) & 1u) == 0) {  // 'h': through the vertical river at x = xhi
      const int y = ylo + 1 + (int)ds.next_bounded((uint32_t)(yhi - ylo - 1));
      g.set(xhi, y, CELL_EMPTY);
      xlo = xhi;
      xhi = next_limit(vmask, xlo, W - 1);
    } else {                        // 'v': through the horizontal river at y = yhi
      const int x = xlo + 1 + (int)ds.next_bounded((uint32_t)(xhi - xlo - 1));
      g.set(x, yhi, CELL_EMPTY);
      ylo = yhi;
      yhi = next_limit(hmask, ylo, H - 1);
    }
  }
}

// WARP: the whole warp calls this for ONE env (same arguments in every lane,
// converged) and KeyCorridor's connect_all runs 32 of its iterations at once
// (see the loop); every other family and step is computed redundantly.
template <int FAM, int H, int W, bool WARP = false>
__device__ __noinline__ GenOut generate_level(RowViewT<Cfg<FAM, H, W>::RW> g, uint32_t genv, uint32_t episode,
                                              uint32_t klo, uint32_t khi, int gparam) {
  using C = Cfg<FAM, H, W>;
  GenOut o{1, 1, 0, 0u, 0u, 0u};
  // the rows are this env's SMEM planes: tell the out-of-line generator so its
  // stores are STS, not generic stores resolved at run time
  __builtin_assume(__isShared(g.rows));
#pragma unroll
  for (int p = 0; p < H * C::RW; ++p) g.rows[p * TILE] = template_plane<FAM, H, W>(p);
  using Draws = typename LevelDrawsT<FAM, WARP>::type;
  Draws ds = make_draws(static_cast<Draws*>(nullptr), genv, episode, klo, khi);

  if constexpr (FAM == FAM_EMPTY_RANDOM) {
    // [MG] EmptyEnv with agent_start_pos=None: place_agent() over the empty
    // cells (the goal is the last interior cell in row-major order, so the
    // admissible set is the first (W-2)(H-2)-1 interior cells), then a direction
    const uint32_t k = ds.next_bounded((uint32_t)((W - 2) * (H - 2) - 1));
    o.ax = 1 + (int)(k % (W - 2));
    o.ay = 1 + (int)(k / (W - 2));
    o.dir = (int)ds.next_bounded(4);
  } else if constexpr (FAM == FAM_FOURROOMS) {
    // [MG] FourRoomsEnv._gen_grid (R#38): one opening per inner wall segment
    // in [MG]'s order (right wall of room (0,0), bottom of (0,0), bottom of
    // (1,0), right of (0,1)); then place_agent() and place_obj(Goal) over the
    // whole grid, uniform over the empty cells in row-major order
    constexpr int RX = W / 2, RY = H / 2;
    const int o0 = 1 + (int)ds.next_bounded(RY - 1);               // (RX, o0)
    const int o1 = 1 + (int)ds.next_bounded(RX - 1);               // (o1, RY)
    const int o2 = RX + 1 + (int)ds.next_bounded(W - 1 - RX - 1);  // (o2, RY)
    const int o3 = RY + 1 + (int)ds.next_bounded(H - 1 - RY - 1);  // (RX, o3)
    g.set(RX, o0, CELL_EMPTY);
    g.set(o1, RY, CELL_EMPTY);
    g.set(o2, RY, CELL_EMPTY);
    g.set(RX, o3, CELL_EMPTY);
    // empty cells of row y as a bit mask over x
    constexpr uint32_t inner = ((1u << (W - 1)) - 1u) & ~1u;
    auto row_free = [&](int y) -> uint32_t {
      if (y == RY) return (1u << o1) | (1u << o2);
      return (y == o0 || y == o3) ? inner : inner & ~(1u << RX);
    };
    auto pick = [&](uint32_t k, int skip_x, int skip_y, int& px, int& py) {
      for (int y = 1; y < H - 1; ++y) {
        uint32_t m = row_free(y);
        if (y == skip_y) m &= ~(1u << skip_x);
        const uint32_t c = __popc(m);
        if (k < c) { px = select64(m, k); py = y; return; }
        k -= c;
      }
    };
    const uint32_t nfree = (uint32_t)((H - 2) * (W - 2) - (W - 2) - (H - 2) + 1 + 4);
    pick(ds.next_bounded(nfree), -1, -1, o.ax, o.ay);
    o.dir = (int)ds.next_bounded(4);
    int gx = 0, gy = 0;
    pick(ds.next_bounded(nfree - 1), o.ax, o.ay, gx, gy);
    g.set(gx, gy, CELL_GOAL);
  } else if constexpr (FAM == FAM_GOTODOOR) {
    // [MG] GoToDoorEnv._gen_grid: room size, walls, 4 door positions, 4
    // distinct colours (one draw over the unused ones, R#37), agent, target
    const int w = 5 + (int)ds.next_bounded((uint32_t)(W - 4));
    const int h = 5 + (int)ds.next_bounded((uint32_t)(H - 4));
    // the wall rectangle as whole 8-byte row planes (the room fits in W <= 8)
    static_assert(C::RW == 1, "GoToDoor kernels are instantiated for widths <= 8");
    {
      const uint64_t in_room = w >= 8 ? ~0ull : (1ull << (8 * w)) - 1;  // bytes x < w
      const uint64_t empty = 0x0101010101010101ull * CELL_EMPTY;
      const uint64_t walls = 0x0101010101010101ull * CELL_WALL;
      const uint64_t side = (0xFFull | (0xFFull << (8 * (w - 1))));  // bytes 0 and w-1
      const uint64_t full = (walls & in_room) | (empty & ~in_room);
      const uint64_t mid = (walls & side) | (empty & ~side);
      constexpr uint64_t in_grid = W >= 8 ? ~0ull : (1ull << (8 * W)) - 1;  // cells x >= W stay 0
#pragma unroll
      for (int y = 0; y < H; ++y) g.rows[y * TILE] = ((y == 0 || y == h - 1) ? full : y < h ? mid : empty) & in_grid;
    }
    const int d0 = 2 + (int)ds.next_bounded((uint32_t)(w - 4));
    const int d1 = 2 + (int)ds.next_bounded((uint32_t)(w - 4));
    const int d2 = 2 + (int)ds.next_bounded((uint32_t)(h - 4));
    const int d3 = 2 + (int)ds.next_bounded((uint32_t)(h - 4));
    uint32_t unused = 0x543210u;  // nibbles: the unused colours in order
    uint32_t cols = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t j = ds.next_bounded((uint32_t)(6 - k));
      cols |= ((unused >> (4 * j)) & 15u) << (4 * k);
      const uint32_t low = unused & ((1u << (4 * j)) - 1u);
      unused = low | ((unused >> (4 * j + 4)) << (4 * j));  // erase nibble j
    }
    g.set(d0, 0, make_cell(K_DOOR_CLOSED, cols & 15));
    g.set(d1, h - 1, make_cell(K_DOOR_CLOSED, (cols >> 4) & 15));
    g.set(0, d2, make_cell(K_DOOR_CLOSED, (cols >> 8) & 15));
    g.set(w - 1, d3, make_cell(K_DOOR_CLOSED, (cols >> 12) & 15));
    const uint32_t k = ds.next_bounded((uint32_t)((w - 2) * (h - 2)));  // place_agent(size=(w, h))
    o.ax = 1 + (int)(k % (w - 2));
    o.ay = 1 + (int)(k / (w - 2));
    o.dir = (int)ds.next_bounded(4);
    const uint32_t t = ds.next_bounded(4);
    const int tx = t == 0 ? d0 : t == 1 ? d1 : t == 2 ? 0 : w - 1;
    const int ty = t == 0 ? 0 : t == 1 ? h - 1 : t == 2 ? d2 : d3;
    o.target = (uint32_t)((tx << 4) | ty);
  } else if constexpr (FAM == FAM_CROSSING) {
    // the Table 8 / 9 crossing counts get a generator with N known at compile
    // time: its 3N - 1 draws come from Philox blocks computed up front
    // (independent chains), each at a compile-time word
    const int N = gparam & 0xff;
    const uint8_t obstacle = (gparam & CROSSING_LAVA) ? CELL_LAVA : CELL_WALL;
    switch (N) {
      case 1: { FixedDraws<1> fd(genv, episode, klo, khi); crossing_level<H, W, 1>(g, fd, 1, obstacle); break; }
      case 2: { FixedDraws<2> fd(genv, episode, klo, khi); crossing_level<H, W, 2>(g, fd, 2, obstacle); break; }
      case 3: { FixedDraws<2> fd(genv, episode, klo, khi); crossing_level<H, W, 3>(g, fd, 3, obstacle); break; }
      case 5: { FixedDraws<4> fd(genv, episode, klo, khi); crossing_level<H, W, 5>(g, fd, 5, obstacle); break; }
      default: crossing_level<H, W, 0>(g, ds, N, obstacle); break;
    }
  } else if constexpr (FAM == FAM_DOORKEY) {
    // [MG] DoorKeyEnv._gen_grid: split, agent pos, agent dir, door row, key pos
    const int split = 2 + (int)ds.next_bounded(W - 4);
    for (int y = 0; y < H; ++y) g.set(split, y, CELL_WALL);
    const uint32_t wid = (uint32_t)(split - 1);
    const uint32_t cnt = wid * (H - 2);          // interior cells left of the wall, all empty
    const uint32_t ka = ds.next_bounded(cnt);
    o.ax = 1 + (int)(ka % wid);
    o.ay = 1 + (int)(ka / wid);
    o.dir = (int)ds.next_bounded(4);
    const int door_y = 1 + (int)ds.next_bounded(W - 3);   // R#24
    g.set(split, door_y, make_cell(K_DOOR_LOCKED, COL_YELLOW));
    uint32_t kk = ds.next_bounded(cnt - 1);
    if (kk >= ka) ++kk;                            // skip the agent cell
    g.set(1 + (int)(kk % wid), 1 + (int)(kk / wid), make_cell(K_KEY, COL_YELLOW));
    o.target = (uint32_t)((split << 4) | door_y);  // the opaque layout, for the visibility table
  } else if constexpr (FAM == FAM_LAVAGAP) {
    // [MG] LavaGapEnv._gen_grid
    const int gx = 2 + (int)ds.next_bounded(W - 4);
    const int gy = 1 + (int)ds.next_bounded(H - 2);
    for (int y = 1; y <= H - 2; ++y)
      if (y != gy) g.set(gx, y, CELL_LAVA);
  } else if constexpr (FAM == FAM_DYNOBS) {
    // [MG] DynamicObstaclesEnv._gen_grid: balls uniform over empty cells, not the agent
    // (free-cell bit y * RS + x, row-major; RS = 8 up to width 8: one word)
    constexpr int RSB = W > 8 ? 16 : 8, NWD = (H * RSB + 63) / 64;
    uint64_t freem[NWD];
#pragma unroll
    for (int w = 0; w < NWD; ++w) freem[w] = 0;
#pragma unroll
    for (int y = 1; y <= H - 2; ++y)
#pragma unroll
      for (int x = 1; x <= W - 2; ++x) freem[(y * RSB + x) >> 6] |= 1ull << ((y * RSB + x) & 63);
    freem[((H - 2) * RSB + (W - 2)) >> 6] &= ~(1ull << (((H - 2) * RSB + (W - 2)) & 63));  // goal
    if (gparam) {
      // Dynamic-Obstacles-Random: place_agent() over the empty cells (the goal
      // is the last interior cell in row-major order), then a direction
      const uint32_t k = ds.next_bounded((uint32_t)((W - 2) * (H - 2) - 1));
      o.ax = 1 + (int)(k % (W - 2));
      o.ay = 1 + (int)(k / (W - 2));
      o.dir = (int)ds.next_bounded(4);
    }
    {
      const int ab = o.ay * RSB + o.ax;  // the agent's cell
#pragma unroll
      for (int w = 0; w < NWD; ++w)
        freem[w] &= ~word_bit(ab, w);
    }
#pragma unroll
    for (int b = 0; b < C::NOBST; ++b) {
      const uint32_t u = ds.next();
      uint32_t cnt = 0;
#pragma unroll
      for (int w = 0; w < NWD; ++w) cnt += __popcll(freem[w]);
      if (cnt == 0) { o.fail += 1; continue; }
      const int pos = select_bits(freem, bounded(u, cnt));
      if constexpr (NWD == 1) freem[0] &= ~(1ull << pos);
      else {
#pragma unroll
        for (int w = 0; w < NWD; ++w) freem[w] &= ~word_bit(pos, w);
      }
      const int x = pos % RSB, y = pos / RSB;
      g.set(x, y, make_cell(K_BALL, COL_BLUE));
      o.balls |= (uint64_t)ball_code(W, x, y) << (8 * b);
    }
  } else if constexpr (FAM == FAM_KEYCORRIDOR) {
    // [MG] RoomGrid._gen_grid + KeyCorridorEnv._gen_grid + connect_all
    constexpr int S = C::RS, NR = C::NR, NC = 3, NROOM = NR * NC;
    // door_pos[0].y (right wall) and door_pos[1].x (bottom wall) per room,
    // drawn room by room (j outer, i inner) as [MG] does
    // nibble r of dpy / dpx = room r's door position (< 16 on grids of at most
    // 17 cells; registers, not a dynamically indexed local array)
    static_assert(H <= 17 && W <= 17 && NROOM <= 16, "door positions are packed in nibbles");
    uint64_t dpy = 0, dpx = 0;
    auto nib = [](uint64_t w, int r) { return (int)((w >> (4 * r)) & 15u); };
    for (int j = 0; j < NR; ++j)
      for (int i = 0; i < NC; ++i) {
        const int r = j * NC + i;
        if (i < NC - 1) dpy |= (uint64_t)(j * (S - 1) + 1 + ds.next_bounded(S - 2)) << (4 * r);
        if (j < NR - 1) dpx |= (uint64_t)(i * (S - 1) + 1 + ds.next_bounded(S - 2)) << (4 * r);
      }
    // room links as bit masks over rooms r = 3j + i: H bit r = rooms r, r+1
    // linked; V bit r = rooms r, r+3 linked (removed walls and doors of any state)
    uint32_t Hl = 0, Vl = 0;
    const int adx = (NC / 2) * (S - 1) + S / 2, ady = (NR / 2) * (S - 1) + S / 2;  // default agent
    // hallway: remove_wall(1, j, up) for j >= 1
    for (int j = 1; j < NR; ++j) {
      for (int t = 1; t < S - 1; ++t) g.set((S - 1) + t, j * (S - 1), CELL_EMPTY);
      Vl |= 1u << ((j - 1) * NC + 1);
    }
    const int room_idx = (int)ds.next_bounded(NR);
    const uint8_t door_col = (uint8_t)ds.next_bounded(6);           // R#23
    const int locked_room = room_idx * NC + 2;
    g.set(2 * (S - 1), nib(dpy, room_idx * NC + 1), make_cell(K_DOOR_LOCKED, door_col));
    Hl |= 1u << (locked_room - 1);
    // object placement inside room (ri, rj): empty, not the default agent
    // cell, Manhattan distance >= 2 from it (reject_next_to, R#25)
    // WARP (the whole warp builds this level): lane l evaluates candidate
    // cell l of a room and ballots assemble the mask, instead of every lane
    // walking all S*S cells (rooms of up to 32 cells)
    constexpr bool LANES = WARP && S * S <= 32;
    const int lane = (int)(threadIdx.x & 31);
    auto place_in_room = [&](int ri, int rj, uint8_t cell) {
      const uint32_t u = ds.next();
      uint64_t m = 0;
      int n = 0;
      if (LANES) {
        const int xx = lane % S, yy = lane / S;
        const int x = ri * (S - 1) + xx, y = rj * (S - 1) + yy;
        const bool ok = lane < S * S && x < W && y < H && g.get(x < W ? x : 0, y < H ? y : 0) == CELL_EMPTY &&
                        abs(x - adx) + abs(y - ady) >= 2;
        m = __ballot_sync(0xffffffffu, ok);
        n = __popc((uint32_t)m);
      } else {
        for (int yy = 0; yy < S; ++yy)
          for (int xx = 0; xx < S; ++xx) {
            const int x = ri * (S - 1) + xx, y = rj * (S - 1) + yy;
            const int d = abs(x - adx) + abs(y - ady);
            const bool ok = x < W && y < H && g.get(x, y) == CELL_EMPTY && d >= 2;
            m |= (ok ? 1ull : 0ull) << (yy * S + xx);
            n += ok;
          }
      }
      if (n == 0) { o.fail += 1; return; }
      const int p = select64(m, bounded(u, (uint32_t)n));
      g.set(ri * (S - 1) + p % S, rj * (S - 1) + p / S, cell);
    };
    const uint8_t ball_col = (uint8_t)ds.next_bounded(6);
    place_in_room(2, room_idx, make_cell(K_BALL, ball_col));
    const int kr = (int)ds.next_bounded(NR);
    place_in_room(0, kr, make_cell(K_KEY, door_col));
    // place_agent(1, NR/2): (pos, dir) uniform over pairs whose front is empty or a wall
    {
      const uint32_t u = ds.next();
      constexpr int NWD = (S * S * 4 + 63) / 64;
      uint64_t m[NWD];
#pragma unroll
      for (int w = 0; w < NWD; ++w) m[w] = 0;
      int n = 0;
      const int rx = S - 1, ry = (NR / 2) * (S - 1);
      if (LANES) {
        // lane c holds candidate cell c's 4 directions as a nibble; the k-th
        // candidate (row-major, direction innermost) is found by prefix counts
        const int xx = lane % S, yy = lane / S, x = rx + xx, y = ry + yy;
        uint32_t nib = 0;
        if (lane < S * S && g.get(x, y) == CELL_EMPTY) {
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const uint8_t f = g.get(x + (d == 0) - (d == 2), y + (d == 1) - (d == 3));
            nib |= (f == CELL_EMPTY || (f & 15) == K_WALL) ? 1u << d : 0u;
          }
        }
        const uint32_t cnt = __popc(nib);
        uint32_t excl = 0;  // candidates in lanes below this one
#pragma unroll
        for (int d = 0; d < 4; ++d)
          excl += __popc(__ballot_sync(0xffffffffu, (nib >> d) & 1u) & ((1u << lane) - 1u));
        const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
        if (total == 0) {
          o.fail += 1;
        } else {
          const uint32_t k = bounded(u, total);
          const int owner = __ffs(__ballot_sync(0xffffffffu, excl <= k && k < excl + cnt)) - 1;
          uint32_t r = __shfl_sync(0xffffffffu, nib, owner);
          const uint32_t kk = k - __shfl_sync(0xffffffffu, excl, owner);  // kk-th set bit of r (kk <= 3)
          r = kk >= 1 ? r & (r - 1u) : r;
          r = kk >= 2 ? r & (r - 1u) : r;
          r = kk >= 3 ? r & (r - 1u) : r;
          o.dir = __ffs(r) - 1;
          o.ax = rx + owner % S;
          o.ay = ry + owner / S;
        }
      } else {
      for (int yy = 0; yy < S; ++yy)
        for (int xx = 0; xx < S; ++xx) {
          const int x = rx + xx, y = ry + yy;
          if (g.get(x, y) != CELL_EMPTY) continue;
          for (int d = 0; d < 4; ++d) {
            const int fx = x + (d == 0) - (d == 2), fy = y + (d == 1) - (d == 3);
            const uint8_t f = g.get(fx, fy);
            const bool ok = f == CELL_EMPTY || (f & 15) == K_WALL;
            const int bit = (yy * S + xx) * 4 + d;
            if constexpr (NWD == 1) m[0] |= (ok ? 1ull : 0ull) << bit;
            else {  // no m[bit >> 6]: a dynamic index puts m in local memory
#pragma unroll
              for (int w = 0; w < NWD; ++w) m[w] |= ok ? word_bit(bit, w) : 0ull;
            }
            n += ok;
          }
        }
      if (n == 0) {
        o.fail += 1;
      } else {
        const int p = select_bits(m, bounded(u, (uint32_t)n));
        o.dir = p & 3;
        o.ax = rx + (p >> 2) % S;
        o.ay = ry + (p >> 2) / S;
      }
      }
    }
    // connect_all(max_itrs = 5000): reachability from the agent's room is kept
    // incrementally (links only grow) and closed bit-parallel over H/V
    const uint32_t all = (1u << NROOM) - 1;
    auto closure = [&](uint32_t reach) {
      uint32_t prev;
      do {
        prev = reach;
        reach |= ((reach & Hl) << 1) | ((reach >> 1) & Hl) | ((reach & Vl) << NC) | ((reach >> NC) & Vl);
      } while (reach != prev);
      return reach;
    };
    uint32_t reach = closure(1u << ((o.ay / (S - 1)) * NC + o.ax / (S - 1)));
    if constexpr (WARP) {
      // The same loop, 32 iterations per round: lane l evaluates iteration
      // it + l as if iterations it .. it + l - 1 were all skips (3 draws
      // each, no state change), i.e. from draw p + 3l.  The first lane that
      // adds a door (or passes the 5000 cap) is the one the sequential loop
      // reaches; its add is applied and the next round starts after its 4th
      // draw.  Same draws, same result, ~#doors + #iterations/32 rounds.
      const uint32_t lane = threadIdx.x & 31;
      uint32_t p = ds.pos;
      int it = 0;
      for (;;) {
        if (it > 5000) { o.fail += 1; break; }
        if (reach == all) break;
        ds.ensure(p >> 2, ((p + 3u * 31u) >> 2) + 2u - (p >> 2));  // this round's <= 26 blocks
        const uint32_t q = p + 3u * lane, b0 = q >> 2, t0 = q & 3;
        const uint4 x0 = ds.block(b0);
        const uint4 x1 = ds.block(b0 + 1u);
        const int i = (int)bounded(pick8(x0, x1, t0), NC);
        const int j = (int)bounded(pick8(x0, x1, t0 + 1), NR);
        const int k = (int)bounded(pick8(x0, x1, t0 + 2), 4);
        const uint32_t wc = pick8(x0, x1, t0 + 3);
        const int r = j * NC + i;
        const bool has = k == 0 ? i < NC - 1 : k == 1 ? j < NR - 1 : k == 2 ? i > 0 : j > 0;
        const int nb = k == 0 ? r + 1 : k == 1 ? r + NC : k == 2 ? r - 1 : r - NC;
        const int lo = r < nb ? r : nb;
        const bool horiz = (k & 1) == 0;
        const bool add = has && !(((horiz ? Hl : Vl) >> lo) & 1u) && r != locked_room && nb != locked_room;
        const uint32_t hit = __ballot_sync(0xffffffffu, add || it + (int)lane > 5000);
        if (hit == 0) { p += 96u; it += 32; continue; }
        const int f = __ffs(hit) - 1;
        it += f;
        if (it > 5000) { o.fail += 1; break; }
        const int fr = __shfl_sync(0xffffffffu, r, f), fnb = __shfl_sync(0xffffffffu, nb, f);
        const int flo = __shfl_sync(0xffffffffu, lo, f);
        const bool fh = __shfl_sync(0xffffffffu, (int)horiz, f) != 0;
        const uint8_t col = (uint8_t)bounded(__shfl_sync(0xffffffffu, wc, f), 6);
        const int li = flo % NC, lj = flo / NC;
        const int x = fh ? li * (S - 1) + S - 1 : nib(dpx, flo);
        const int y = fh ? nib(dpy, flo) : lj * (S - 1) + S - 1;
        g.set(x, y, make_cell(K_DOOR_CLOSED, col));
        if (fh) Hl |= 1u << flo;
        else Vl |= 1u << flo;
        if (((reach >> fr) ^ (reach >> fnb)) & 1u) reach = closure(reach);
        p += 3u * (uint32_t)f + 4u;
        it += 1;
      }
      return o;
    }
    for (int it = 0;; ++it) {
      if (it > 5000) { o.fail += 1; break; }
      if (reach == all) break;
      const int i = (int)ds.next_bounded(NC);
      const int j = (int)ds.next_bounded(NR);
      const int k = (int)ds.next_bounded(4);
      const int r = j * NC + i;
      const bool has = k == 0 ? i < NC - 1 : k == 1 ? j < NR - 1 : k == 2 ? i > 0 : j > 0;
      if (!has) continue;
      const int nb = k == 0 ? r + 1 : k == 1 ? r + NC : k == 2 ? r - 1 : r - NC;
      const int lo = r < nb ? r : nb;  // the link's lower room: its door_pos[0] or door_pos[1]
      const bool horiz = (k & 1) == 0;
      if ((((horiz ? Hl : Vl) >> lo) & 1u)) continue;
      if (r == locked_room || nb == locked_room) continue;
      const uint8_t col = (uint8_t)ds.next_bounded(6);
      const int li = lo % NC, lj = lo / NC;
      const int x = horiz ? li * (S - 1) + S - 1 : nib(dpx, lo);
      const int y = horiz ? nib(dpy, lo) : lj * (S - 1) + S - 1;
      g.set(x, y, make_cell(K_DOOR_CLOSED, col));
      if (horiz) Hl |= 1u << lo;
      else Vl |= 1u << lo;
      if (((reach >> r) ^ (reach >> nb)) & 1u) reach = closure(reach);
    }
  }
  return o;
}

}  // namespace navix
