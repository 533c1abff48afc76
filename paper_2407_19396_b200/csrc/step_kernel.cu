// step_kernel.cu — the fused batched MiniGrid step for sm_100a.
//
// One thread owns one environment; one CTA owns a tile of TILE = 128 envs.
// Per env and step:
//   a1 stage      coalesced 64-bit loads of the H grid row planes + agent record
//                 into SMEM row lines (struct-of-arrays, layout.h)
//   a2 autoreset  if the previous step ended: episode += 1, Philox level
//                 generation into the SMEM rows (levelgen.cuh), first obs
//   a3 transition Dynamic-Obstacles balls (Table 3, App. A)
//   a4 intervene  left/right/forward/pickup/drop/toggle/done
//   a5 reward     Eq. (1) P:216 / P:223 (R#1-R#3), events -> terminated,
//                 step_count >= T -> truncated (R#17)
//   a6 observe    symbolic_first_person (Table 5): the 7 view columns
//                 are 7 world lines (rows or columns, read from SMEM row /
//                 column copies) shifted and byte-reversed; MiniGrid's
//                 process_vis as 7-bit row closures computed with one
//                 integer add each (carry = propagation); SWAR encode of 4
//                 cells per 32-bit word; interleave (type, colour, state) with
//                 byte permutes; the 147-byte record assembled in registers
//   a7 store      obs staged in SMEM, written by ONE cp.async.bulk (TMA bulk
//                 copy) per tile; reward/flags/agent records coalesced;
//                 grid rows written back only when modified; episode
//                 statistics warp-reduced into striped int64 counters.
#include <cstdint>

#include "layout.h"
#include "levelgen.cuh"
#include "philox.cuh"

namespace navix {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8x8 byte transpose: rows r[y] (byte x) -> cols c[x] (byte y), 32 byte permutes.
__device__ __forceinline__ void transpose4x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& o0,
                                             uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o0 = __byte_perm(t0, t1, 0x5410);
  o1 = __byte_perm(t0, t1, 0x7632);
  o2 = __byte_perm(t2, t3, 0x5410);
  o3 = __byte_perm(t2, t3, 0x7632);
}

template <int H, int W>
__device__ __forceinline__ void build_cols(const uint64_t* rows, uint64_t* cols) {
  uint32_t lo[8], hi[8];
#pragma unroll
  for (int y = 0; y < 8; ++y) {
    const uint64_t r = y < H ? rows[y * TILE] : 0ull;
    lo[y] = (uint32_t)r;
    hi[y] = (uint32_t)(r >> 32);
  }
  uint32_t a[4], b[4], c[4], d[4];
  transpose4x4(lo[0], lo[1], lo[2], lo[3], a[0], a[1], a[2], a[3]);  // x 0..3, y 0..3
  transpose4x4(lo[4], lo[5], lo[6], lo[7], b[0], b[1], b[2], b[3]);  // x 0..3, y 4..7
  transpose4x4(hi[0], hi[1], hi[2], hi[3], c[0], c[1], c[2], c[3]);  // x 4..7, y 0..3
  transpose4x4(hi[4], hi[5], hi[6], hi[7], d[0], d[1], d[2], d[3]);  // x 4..7, y 4..7
#pragma unroll
  for (int x = 0; x < W; ++x) {
    const uint64_t v = x < 4 ? ((uint64_t)b[x] << 32) | a[x] : ((uint64_t)d[x - 4] << 32) | c[x - 4];
    cols[x * TILE] = v;
  }
}

// SWAR encode of 4 cells: (type, colour, state) bytes, masked by visibility.
__device__ __forceinline__ void encode4(uint32_t w, uint32_t m, uint32_t& ty, uint32_t& co, uint32_t& st) {
  const uint32_t E = w & 0x0F0F0F0Fu;
  co = ((w >> 4) & 0x07070707u) & m;
  const uint32_t ge = (E + 0x05050505u) & 0x10101010u;  // kind >= 11: closed / locked door
  const uint32_t d = ge >> 4;
  const uint32_t dm = ge - d;                            // 0x0F per door byte
  ty = ((E & ~dm) | (d << 2)) & m;                       // doors -> 4
  st = ((E & dm) - d * 10u) & m;                         // 11 -> 1, 12 -> 2
}

// Interleave 4 cells' (t, c, s) bytes into 12 bytes (3 words).
__device__ __forceinline__ void interleave4(uint32_t ty, uint32_t co, uint32_t st, uint32_t& q0, uint32_t& q1,
                                            uint32_t& q2) {
  const uint32_t x0 = __byte_perm(ty, co, 0x5140);  // t0 c0 t1 c1
  const uint32_t x1 = __byte_perm(ty, co, 0x7362);  // t2 c2 t3 c3
  q0 = __byte_perm(x0, st, 0x2410);                 // t0 c0 s0 t1
  const uint32_t y = __byte_perm(x0, st, 0x0053);   // c1 s1 .  .
  q1 = __byte_perm(y, x1, 0x5410);                  // c1 s1 t2 c2
  q2 = __byte_perm(x1, st, 0x7326);                 // s2 t3 c3 s3
}

// Place the 21-byte column VI at byte 21*VI of the 147-byte record.
template <int VI>
__device__ __forceinline__ void emit_column(uint32_t (&rec)[37], const uint32_t (&w)[6]) {
  constexpr int O = 21 * VI, B = O / 4, R = O % 4;
  if constexpr (R == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) rec[B + k] = w[k];
  } else {
    rec[B] |= w[0] << (8 * R);
#pragma unroll
    for (int k = 1; k < 6; ++k) rec[B + k] = __funnelshift_l(w[k - 1], w[k], 8 * R);
  }
}

// The egocentric view column VI (lateral offset VI-3) as 7 cell bytes
// (byte vj = distance 6-vj from the agent): a window of one world line.
struct ViewGeom {
  const uint64_t* lines;  // &s_rows[0][tid] or &s_cols[0][tid]
  int base, sgn, nlines, shift, rev;
};

__device__ __forceinline__ uint64_t view_column(const ViewGeom& g, int vi) {
  const int L = g.base + g.sgn * vi;
  uint64_t line = 0;
  if ((unsigned)L < (unsigned)g.nlines) line = g.lines[L * TILE];
  uint64_t wv = g.shift >= 0 ? (line >> (8 * g.shift)) : (line << (-8 * g.shift));
  wv &= 0x00FFFFFFFFFFFFFFull;
  const uint32_t lo = (uint32_t)wv, hi = (uint32_t)(wv >> 32);
  const uint64_t rv = ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32 | __byte_perm(hi, 0, 0x0123)) >> 8;
  return g.rev ? rv : wv;
}

template <int VI>
__device__ __forceinline__ void encode_column(uint32_t (&rec)[37], uint64_t colv, uint64_t vis) {
  const uint64_t m = ((vis >> VI) & 0x0101010101010101ull) * 0xFFull;
  uint32_t ty, co, st, w[6];
  encode4((uint32_t)colv, (uint32_t)m, ty, co, st);
  interleave4(ty, co, st, w[0], w[1], w[2]);
  encode4((uint32_t)(colv >> 32), (uint32_t)(m >> 32), ty, co, st);
  uint32_t unused;
  interleave4(ty, co, st, w[3], w[4], unused);
  w[5] = (st >> 16) & 0xFFu;  // s6
  emit_column<VI>(rec, w);
}

// a6: the 147-byte observation of one env (Table 5, [MG] gen_obs).
template <int H, int W>
__device__ __forceinline__ void observe(const uint64_t* rows, const uint64_t* cols, int ax, int ay, int dir,
                                        uint8_t carry, uint32_t (&rec)[37]) {
  // view column vi <-> world line parallel to the facing direction:
  //  dir 0 (east):  row    ay+vi-3, x = ax+6-vj  (reversed window from ax)
  //  dir 1 (south): column ax+3-vi, y = ay+6-vj  (reversed window from ay)
  //  dir 2 (west):  row    ay+3-vi, x = ax-6+vj  (window from ax-6)
  //  dir 3 (north): column ax+vi-3, y = ay-6+vj  (window from ay-6)
  ViewGeom g;
  const bool odd = dir & 1;
  g.lines = odd ? cols : rows;
  g.nlines = odd ? W : H;
  g.base = dir == 0 ? ay - 3 : dir == 1 ? ax + 3 : dir == 2 ? ay + 3 : ax - 3;
  g.sgn = (dir == 0 || dir == 3) ? 1 : -1;
  g.shift = dir == 0 ? ax : dir == 1 ? ay : dir == 2 ? ax - 6 : ay - 6;
  g.rev = dir <= 1;
  uint64_t col[7];
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) col[vi] = view_column(g, vi);
  // opacity rows: byte vj of OP has bit vi set iff view cell (vi, vj) is opaque
  uint64_t op = 0;
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) op |= (col[vi] & 0x8080808080808080ull) >> (7 - vi);
  // [MG] process_vis: rows vj = 6 .. 0; within a row the visible set is the
  // closure of the seeds; a rightward closure is the carry chain of
  // T + (T & S) (carry into bit k = "k-1 visible and transparent"), the
  // leftward one the same on bit-reversed rows.
  uint64_t vis = 0;
  uint32_t seed = 1u << 3;
#pragma unroll
  for (int j = 6; j >= 0; --j) {
    const uint32_t t = ~(uint32_t)(op >> (8 * j)) & 0x7Fu;
    uint32_t ts = t & seed;
    uint32_t v = (seed | ((t + ts) ^ t ^ ts)) & 0x7Fu;
    const uint32_t tr = __brev(t) >> 25;
    uint32_t vr = __brev(v) >> 25;
    ts = tr & vr;
    vr = (vr | ((tr + ts) ^ tr ^ ts)) & 0x7Fu;
    v = __brev(vr) >> 25;
    const uint32_t a = v & t;
    seed = (a | (a << 1) | (a >> 1)) & 0x7Fu;
    vis |= (uint64_t)v << (8 * j);
  }
  // the agent sees what it carries (R#13): view cell (3, 6)
  col[3] = (col[3] & ~(0xFFull << 48)) | ((uint64_t)carry << 48);
  encode_column<0>(rec, col[0], vis);
  encode_column<1>(rec, col[1], vis);
  encode_column<2>(rec, col[2], vis);
  encode_column<3>(rec, col[3], vis);
  encode_column<4>(rec, col[4], vis);
  encode_column<5>(rec, col[5], vis);
  encode_column<6>(rec, col[6], vis);
}

// Store the 147-byte record at byte tid*147 of the SMEM staging buffer.
__device__ __forceinline__ void stage_obs(uint8_t* s_obs, int tid, const uint32_t (&rec)[37]) {
  const uint32_t off = (uint32_t)tid * OBS_BYTES;
  const uint32_t m = off & 3u, sh = 8u * m;
  uint32_t* s32 = reinterpret_cast<uint32_t*>(s_obs) + (off >> 2);
  uint8_t* s8 = reinterpret_cast<uint8_t*>(s32);
  const uint32_t first = rec[0] << sh;
  if (m == 0) s32[0] = first;
  else if (m == 1) { s8[1] = (uint8_t)(first >> 8); *reinterpret_cast<uint16_t*>(s8 + 2) = (uint16_t)(first >> 16); }
  else if (m == 2) *reinterpret_cast<uint16_t*>(s8 + 2) = (uint16_t)(first >> 16);
  else s8[3] = (uint8_t)(first >> 24);
#pragma unroll
  for (int j = 1; j < 36; ++j) s32[j] = __funnelshift_l(rec[j - 1], rec[j], sh);
  const uint32_t w36 = __funnelshift_l(rec[35], rec[36], sh);
  if (m >= 1) s32[36] = w36;
  else { *reinterpret_cast<uint16_t*>(s8 + 144) = (uint16_t)w36; s8[146] = (uint8_t)(w36 >> 16); }
  const uint32_t w37 = __funnelshift_l(rec[36], 0u, sh);
  if (m == 2) s8[148] = (uint8_t)w37;
  else if (m == 3) *reinterpret_cast<uint16_t*>(s8 + 148) = (uint16_t)w37;
}

__device__ __forceinline__ float success_reward(int mode, uint32_t sc, uint32_t T) {
  if (mode == 1) return 1.0f;
  // R#2: binary64, [MG] order, no contraction, one rounding to binary32
  const double q = __ddiv_rn((double)sc, (double)T);
  const double p = __dmul_rn(0.9, q);
  return __double2float_rn(__dsub_rn(1.0, p));
}

// ------------------------------------------------------------------ kernel
template <int FAM, int H, int W, int MODE>
__global__ void __launch_bounds__(TILE) navix_kernel(const KernelArgs a) {
  using C = Cfg<FAM, H, W>;
  __shared__ __align__(128) uint8_t s_obs[TILE * OBS_BYTES];
  __shared__ __align__(16) uint64_t s_rows[H][TILE];
  __shared__ __align__(16) uint64_t s_cols[W][TILE];
  __shared__ unsigned int s_any;

  const int tid = threadIdx.x;
  const int64_t e = (int64_t)blockIdx.x * TILE + tid;
  const bool valid = e < a.n;
  const uint32_t genv = a.env_begin + (uint32_t)e;
  uint64_t* const rows = &s_rows[0][tid];
  uint64_t* const cols = &s_cols[0][tid];
  RowView g{rows};

  // ---- a1: stage
  uint8_t act = 0;
  uint64_t rec = 0;
  uint32_t balls = 0, episode = 0;
  if (MODE != MODE_RESET) {
    const uint64_t* gsrc = a.grid + (int64_t)blockIdx.x * H * TILE + tid;
#pragma unroll
    for (int y = 0; y < H; ++y) rows[y * TILE] = gsrc[y * TILE];
    rec = a.agent[e];
    if (MODE == MODE_STEP && valid) act = a.actions[e];
    if (FAM == FAM_DYNOBS) {
      balls = a.balls[e];
      if (MODE == MODE_STEP) episode = a.episode[e];
    }
  }
  int ax = (int)(rec & 0xFF), ay = (int)((rec >> 8) & 0xFF), dir = (int)((rec >> 16) & 3);
  uint8_t carry = (uint8_t)(rec >> 24);
  uint32_t sc = (uint32_t)((rec >> 32) & 0xFFFF);
  bool prev_done = (rec >> 48) & 1;

  float reward = 0.f;
  bool term = false, trunc = false, grid_dirty = false;
  uint32_t st_ep = 0, st_len = 0, st_succ = 0, st_succ_len = 0, st_lava = 0, st_coll = 0, st_trunc = 0,
           st_fail = 0;

  const bool regen = MODE == MODE_RESET || (MODE == MODE_STEP && prev_done);
  if (regen) {
    // ---- a2: next-step auto-reset (R#18) / reset(key)
    if (MODE == MODE_STEP) {
      if (FAM != FAM_DYNOBS) episode = a.episode[e];
      episode += 1;
    }
    const GenOut o = generate_level<FAM, H, W>(g, genv, episode, a.key_lo, a.key_hi);
    ax = o.ax; ay = o.ay; dir = o.dir;
    balls = o.balls;
    st_fail = o.fail;
    carry = CELL_EMPTY;
    sc = 0;
    prev_done = false;
    grid_dirty = true;
  } else {
    if (FAM == FAM_DYNOBS) {
#pragma unroll
      for (int b = 0; b < C::NOBST; ++b) {
        const uint32_t p = (balls >> (8 * b)) & 0xFF;
        if (p) g.set(p >> 4, p & 15, make_cell(K_BALL, COL_BLUE));
      }
    }
    if (MODE == MODE_STEP) {
      const int dx = dir == 0 ? 1 : dir == 2 ? -1 : 0;
      const int dy = dir == 1 ? 1 : dir == 3 ? -1 : 0;
      const int fx = ax + dx, fy = ay + dy;
      bool not_clear = false;
      if (FAM == FAM_DYNOBS) {
        // ---- a3: transition mu (R#4, R#5, R#7)
        if (act >= 3) act = 0;
        const uint8_t f0 = g.get(fx, fy);
        not_clear = f0 != CELL_EMPTY && (f0 & 15) != K_GOAL;
        const uint4 u = philox4x32_10(make_uint4(genv, episode, (1u << 16) | sc, 0u), a.key_lo, a.key_hi);
#pragma unroll
        for (int b = 0; b < C::NOBST; ++b) {
          const uint32_t p = (balls >> (8 * b)) & 0xFF;
          if (!p) continue;
          const int bx = p >> 4, by = p & 15;
          uint32_t m = 0;
#pragma unroll
          for (int k = 0; k < 9; ++k) {
            const int x = bx - 1 + k % 3, y = by - 1 + k / 3;
            const bool ok = g.get(x, y) == CELL_EMPTY && !(x == ax && y == ay);
            m |= (ok ? 1u : 0u) << k;
          }
          if (m) {
            const uint32_t ub = b == 0 ? u.x : b == 1 ? u.y : b == 2 ? u.z : u.w;
            const int k = select64(m, bounded(ub, __popc(m)));
            const int nx = bx - 1 + k % 3, ny = by - 1 + k / 3;
            g.set(nx, ny, make_cell(K_BALL, COL_BLUE));
            g.set(bx, by, CELL_EMPTY);
            balls = (balls & ~(0xFFu << (8 * b))) | ((uint32_t)((nx << 4) | ny) << (8 * b));
          }
        }
      }
      // ---- a4: intervention I (Table 3; [MG] MiniGridEnv.step)
      sc += 1;
      uint8_t* fp = g.at(fx, fy);
      const uint8_t fc = *fp;
      const uint32_t kind = fc & 15u;
      bool success = false, lava = false, coll = false;
      switch (act) {
        case 0: dir = (dir + 3) & 3; break;
        case 1: dir = (dir + 1) & 3; break;
        case 2:
          if ((0x31Au >> kind) & 1u) { ax = fx; ay = fy; }  // empty, floor, open door, goal, lava
          success = kind == K_GOAL;
          lava = kind == K_LAVA;
          break;
        case 3:
          if (((0xE0u >> kind) & 1u) && carry == CELL_EMPTY) {  // key, ball, box
            carry = fc;
            *fp = CELL_EMPTY;
            grid_dirty = true;
          }
          break;
        case 4:
          if (fc == CELL_EMPTY && carry != CELL_EMPTY) {
            *fp = carry;
            carry = CELL_EMPTY;
            grid_dirty = true;
          }
          break;
        case 5: {
          const uint8_t col = (fc >> 4) & 7;
          if (kind == K_DOOR_LOCKED) {
            if ((carry & 15) == K_KEY && ((carry >> 4) & 7) == col) {
              *fp = make_cell(K_DOOR_OPEN, col);
              grid_dirty = true;
            }
          } else if (kind == K_DOOR_CLOSED) {
            *fp = make_cell(K_DOOR_OPEN, col);
            grid_dirty = true;
          } else if (kind == K_DOOR_OPEN) {
            *fp = make_cell(K_DOOR_CLOSED, col);
            grid_dirty = true;
          } else if (kind == K_BOX) {
            *fp = CELL_EMPTY;
            grid_dirty = true;
          }
          break;
        }
        default: break;  // done, and out-of-range actions (R#15)
      }
      if (FAM == FAM_KEYCORRIDOR && act == 3 && (carry & 15) == K_BALL) success = true;  // R#8
      if (FAM == FAM_DYNOBS && act == 2 && not_clear) { coll = true; success = false; }  // R#4
      // ---- a5: reward and termination (Eq. 1, Tables 6-7)
      if (coll) reward = -1.0f;
      else if (success) reward = success_reward(a.reward_mode, sc, C::T);
      else if (lava) reward = a.reward_mode == 1 ? -1.0f : 0.0f;
      term = success || lava || coll;
      trunc = sc >= (uint32_t)C::T && !term;
      prev_done = term || trunc;
      if (prev_done) {
        st_ep = 1;
        st_len = sc;
        st_succ = success;
        st_succ_len = success ? sc : 0;
        st_lava = lava;
        st_coll = coll;
        st_trunc = trunc;
      }
    }
  }

  // ---- a6: observation
  build_cols<H, W>(rows, cols);
  uint32_t obsrec[37];
  observe<H, W>(rows, cols, ax, ay, dir, carry, obsrec);
  stage_obs(s_obs, tid, obsrec);

  // ---- a7: stores
  const int64_t tile_env0 = (int64_t)blockIdx.x * TILE;
  const int64_t nvalid64 = a.n - tile_env0;
  const int nvalid = nvalid64 >= TILE ? TILE : (int)nvalid64;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const bool bulk = a.bulk_obs && nvalid == TILE;
  if (bulk) {
    if (tid == 0) {
      uint8_t* dst = a.obs + tile_env0 * OBS_BYTES;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"(smem_u32(s_obs)), "r"((uint32_t)(TILE * OBS_BYTES))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else {
    uint8_t* dst = a.obs + tile_env0 * OBS_BYTES;
    for (int i = tid; i < nvalid * OBS_BYTES; i += TILE) dst[i] = s_obs[i];
  }

  if (MODE != MODE_OBSERVE) {
    if (valid) {
      if (MODE == MODE_STEP) {
        a.reward[e] = reward;
        a.terminated[e] = term;
        a.truncated[e] = trunc;
      }
      const uint64_t nrec = (uint64_t)(uint32_t)ax | ((uint64_t)(uint32_t)ay << 8) | ((uint64_t)dir << 16) |
                            ((uint64_t)carry << 24) | ((uint64_t)sc << 32) | ((uint64_t)(prev_done ? 1 : 0) << 48);
      a.agent[e] = nrec;
      if (regen) a.episode[e] = episode;
      if (FAM == FAM_DYNOBS) a.balls[e] = balls;
    }
    if (grid_dirty) {
      uint64_t* gdst = a.grid + (int64_t)blockIdx.x * H * TILE + tid;
#pragma unroll
      for (int y = 0; y < H; ++y)
        gdst[y * TILE] = FAM == FAM_DYNOBS ? template_row<FAM, H, W>(y) : rows[y * TILE];
    }
    // episode statistics (info i_{t+1}): warp reduce -> striped atomics
    {
      const unsigned any = __any_sync(0xffffffffu, (st_ep | st_fail) != 0 && valid);
      if (any) {
        const uint32_t vv = valid ? 1u : 0u;
        uint32_t v[8] = {st_ep * vv, st_len * vv, st_succ * vv, st_succ_len * vv,
                         st_lava * vv, st_coll * vv, st_trunc * vv, st_fail * vv};
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __reduce_add_sync(0xffffffffu, v[k]);
        if ((tid & 31) == 0) {
          unsigned long long* slot = a.stats + (size_t)((blockIdx.x * (TILE / 32) + (tid >> 5)) % NSLOT) * 8;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (v[k]) atomicAdd(slot + k, (unsigned long long)v[k]);
        }
      }
    }
  }
  if (bulk && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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

// ------------------------------------------------------------------ dispatch
template <int FAM, int H, int W>
static cudaError_t launch_fhw(int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s) {
  const dim3 grid((unsigned)n_tiles), block(TILE);
  if (mode == MODE_STEP) navix_kernel<FAM, H, W, MODE_STEP><<<grid, block, 0, s>>>(a);
  else if (mode == MODE_RESET) navix_kernel<FAM, H, W, MODE_RESET><<<grid, block, 0, s>>>(a);
  else navix_kernel<FAM, H, W, MODE_OBSERVE><<<grid, block, 0, s>>>(a);
  return cudaPeekAtLastError();
}

cudaError_t launch_env_kernel(const EnvConfig& c, int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s) {
  const int key = c.family * 10000 + c.height * 100 + c.width;
  switch (key) {
    case FAM_EMPTY * 10000 + 505: return launch_fhw<FAM_EMPTY, 5, 5>(mode, a, n_tiles, s);
    case FAM_EMPTY * 10000 + 606: return launch_fhw<FAM_EMPTY, 6, 6>(mode, a, n_tiles, s);
    case FAM_EMPTY * 10000 + 808: return launch_fhw<FAM_EMPTY, 8, 8>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 505: return launch_fhw<FAM_DOORKEY, 5, 5>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 606: return launch_fhw<FAM_DOORKEY, 6, 6>(mode, a, n_tiles, s);
    case FAM_DOORKEY * 10000 + 808: return launch_fhw<FAM_DOORKEY, 8, 8>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 505: return launch_fhw<FAM_DYNOBS, 5, 5>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 606: return launch_fhw<FAM_DYNOBS, 6, 6>(mode, a, n_tiles, s);
    case FAM_DYNOBS * 10000 + 808: return launch_fhw<FAM_DYNOBS, 8, 8>(mode, a, n_tiles, s);
    case FAM_LAVAGAP * 10000 + 505: return launch_fhw<FAM_LAVAGAP, 5, 5>(mode, a, n_tiles, s);
    case FAM_LAVAGAP * 10000 + 606: return launch_fhw<FAM_LAVAGAP, 6, 6>(mode, a, n_tiles, s);
    case FAM_LAVAGAP * 10000 + 707: return launch_fhw<FAM_LAVAGAP, 7, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 307: return launch_fhw<FAM_KEYCORRIDOR, 3, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 507: return launch_fhw<FAM_KEYCORRIDOR, 5, 7>(mode, a, n_tiles, s);
    case FAM_KEYCORRIDOR * 10000 + 707: return launch_fhw<FAM_KEYCORRIDOR, 7, 7>(mode, a, n_tiles, s);
    default: return cudaErrorInvalidConfiguration;
  }
}

cudaError_t launch_sample_actions(uint8_t* out, int64_t n, int64_t steps, uint32_t env_begin, uint32_t t0,
                                  uint64_t seed, uint32_t n_actions, cudaStream_t s) {
  const int64_t total = n * steps;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
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
