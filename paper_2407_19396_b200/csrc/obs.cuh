// obs.cuh — a6, the observation O = symbolic_first_person (Table 5),
// MiniGrid's gen_obs_grid + process_vis + encode (R#10-R#14).
//
// Per env, all in registers + 16 SMEM line loads:
//  1. view column vi (lateral offset vi-3) is a window of ONE world line
//     (a row for dir 0/2, a column for dir 1/3) read with one 64-bit LDS;
//     the shift and the byte reversal of the window are a single byte
//     permute with a per-env selector (out-of-grid positions read arbitrary
//     bytes: with a closed wall border they can never become visible, R#12).
//  2. the 7x7 opacity matrix is gathered as 7 row masks (bit 7 of each cell).
//  3. process_vis as 7 row closures.  Within a row the closure of the seeds
//     is R(S) u L(S): R is the carry chain of T + (T & S) (carry into bit k =
//     "k-1 visible and transparent"), L the same on bit-reversed rows; both
//     run in one 32-bit add on [row | reversed row] with a stopper bit.
//  4. invisible cells are zeroed, the visible ones SWAR-encoded 4 per word to
//     (type, colour, state), and the 147-byte record is assembled with byte
//     permutes at its final byte alignment, which is warp-uniform (a warp
//     owns envs with equal index mod 4), then stored to SMEM word by word.
#pragma once
#include <cstdint>

#include "layout.h"

namespace navix {

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;  // default mode: selector nibble bit 3 replicates the sign of the byte
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// SWAR encode of 4 cell bytes w with visibility byte mask m (0xFF visible,
// 0x00 invisible -> (0,0,0)) to MiniGrid (type, colour, state):
// kind >= 11 (closed 11 / locked 12 door) -> type 4, state kind-10; otherwise
// type = kind, state 0; colour = bits 4-6.  E + 0x75 sets bit 7 of a byte iff
// kind >= 11, and a sign-replicating byte permute turns it into a 0xFF mask.
__device__ __forceinline__ void encode4(uint32_t w, uint32_t m, uint32_t& ty, uint32_t& co, uint32_t& st) {
  const uint32_t E = w & m & 0x0F0F0F0Fu;
  co = (w >> 4) & m & 0x07070707u;
  uint32_t D;
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(D) : "r"(E + 0x75757575u));
  ty = (E & ~D) | (D & 0x04040404u);
  st = (E + 0x06060606u) & D & 0x0F0F0F0Fu;  // (kind + 16 - 10) mod 16, no borrow between bytes
}

// ---------------------------------------------------------------- emission plan
// A column's 21 record bytes (t c s for vj = 0..6) come from 6 registers:
// 0: X00 = (t0 c0 t1 c1)  1: X01 = (t2 c2 t3 c3)  2: S0 = (s0 s1 s2 s3)
// 3: X10 = (t4 c4 t5 c5)  4: X11 = (t6 c6 . .)     5: S1 = (s4 s5 s6 .)
// and register 6 holds the pending partial word of the previous column.
__host__ __device__ constexpr int col_reg(int i) {
  return (i % 3 == 2) ? ((i / 3) / 4 ? 5 : 2) : ((i / 3) / 4) * 3 + ((i / 3) % 4) / 2;
}
__host__ __device__ constexpr int col_byte(int i) {
  return (i % 3 == 2) ? (i / 3) % 4 : 2 * (((i / 3) % 4) % 2) + (i % 3);
}

struct WordPlan {
  int ns;          // distinct sources (1..3)
  int s0, s1, s2;  // source registers
  uint32_t sel0;   // prmt(s0, s1, sel0)
  uint32_t sel1;   // if ns == 3: prmt(tmp, s2, sel1)
};

// Output word k (from the word-aligned record base) of column VI at record
// misalignment M.  Bytes before the column come from the pending word (reg 6),
// bytes after it are don't-care (filled by the next column).
__host__ __device__ constexpr WordPlan plan_word(int M, int VI, int k) {
  int reg[4] = {-1, -1, -1, -1}, byt[4] = {0, 0, 0, 0};
  const int O = M + 21 * VI;
  for (int p = 0; p < 4; ++p) {
    const int i = 4 * k + p - O;
    if (i < 0) {
      if (VI > 0) { reg[p] = 6; byt[p] = p; }
    } else if (i <= 20) {
      reg[p] = col_reg(i);
      byt[p] = col_byte(i);
    }
  }
  int src[3] = {-1, -1, -1}, ns = 0;
  for (int p = 0; p < 4; ++p) {
    if (reg[p] < 0) continue;
    bool seen = false;
    for (int q = 0; q < ns; ++q) seen = seen || src[q] == reg[p];
    if (!seen) src[ns++] = reg[p];
  }
  WordPlan P{ns, src[0], src[1] < 0 ? src[0] : src[1], src[2], 0u, 0u};
  uint32_t s0 = 0, s1 = 0;
  for (int p = 0; p < 4; ++p) {
    uint32_t n0 = 0, n1 = p;  // don't-care bytes: any index
    if (reg[p] == src[0]) { n0 = byt[p]; n1 = p; }
    else if (ns >= 2 && reg[p] == src[1]) { n0 = 4 + byt[p]; n1 = p; }
    else if (ns == 3 && reg[p] == src[2]) { n0 = 0; n1 = 4 + byt[p]; }
    s0 |= n0 << (4 * p);
    s1 |= n1 << (4 * p);
  }
  P.sel0 = s0;
  P.sel1 = s1;
  return P;
}

// Stores bytes [p0, p1] of word v at SMEM word address w (p0 <= p1).
__device__ __forceinline__ void sts_bytes(uint32_t* w, uint32_t v, int p0, int p1) {
  uint8_t* b = reinterpret_cast<uint8_t*>(w);
  if (p0 == 0 && p1 == 3) { *w = v; return; }
  for (int p = p0; p <= p1;) {
    if ((p & 1) == 0 && p + 1 <= p1) {
      *reinterpret_cast<uint16_t*>(b + p) = (uint16_t)(v >> (8 * p));
      p += 2;
    } else {
      b[p] = (uint8_t)(v >> (8 * p));
      p += 1;
    }
  }
}

template <int M, int VI, int K>
__device__ __forceinline__ void emit_word(uint32_t* out, const uint32_t (&r)[7], uint32_t& pend) {
  constexpr WordPlan P = plan_word(M, VI, K);
  uint32_t v;
  if constexpr (P.ns == 3) {
    const uint32_t t = prmt(r[P.s0], r[P.s1], P.sel0);
    v = prmt(t, r[P.s2], P.sel1);
  } else {
    v = prmt(r[P.s0], r[P.s1], P.sel0);
  }
  constexpr int O = M + 21 * VI;
  constexpr int first = 4 * K, last = 4 * K + 3;   // stream bytes covered by word K
  constexpr int col_end = O + 20;                  // last stream byte of this column
  constexpr int rec_end = M + 146;                 // last stream byte of the record
  if constexpr (last <= col_end) {
    // word complete: store (partially if it starts before the record)
    if constexpr (first < M) sts_bytes(out + K, v, M, 3);
    else *(out + K) = v;
  } else if constexpr (col_end == rec_end) {
    sts_bytes(out + K, v, 0, col_end - first);   // record tail
  } else {
    pend = v;                                      // continues in the next column
  }
}

template <int M, int VI>
__device__ __forceinline__ void emit_column(uint32_t* out, const uint32_t (&r)[7], uint32_t& pend) {
  constexpr int O = M + 21 * VI;
  constexpr int K0 = O / 4, K1 = (O + 20) / 4;
  emit_word<M, VI, K0>(out, r, pend);
  emit_word<M, VI, K0 + 1>(out, r, pend);
  emit_word<M, VI, K0 + 2>(out, r, pend);
  emit_word<M, VI, K0 + 3>(out, r, pend);
  emit_word<M, VI, K0 + 4>(out, r, pend);
  if constexpr (K1 >= K0 + 5) emit_word<M, VI, K0 + 5>(out, r, pend);
}

template <int M>
__device__ __forceinline__ void emit_record(uint32_t* out, uint32_t (&r)[7][7]) {
  uint32_t pend = 0;
  r[0][6] = pend;
  emit_column<M, 0>(out, r[0], pend);
  r[1][6] = pend;
  emit_column<M, 1>(out, r[1], pend);
  r[2][6] = pend;
  emit_column<M, 2>(out, r[2], pend);
  r[3][6] = pend;
  emit_column<M, 3>(out, r[3], pend);
  r[4][6] = pend;
  emit_column<M, 4>(out, r[4], pend);
  r[5][6] = pend;
  emit_column<M, 5>(out, r[5], pend);
  r[6][6] = pend;
  emit_column<M, 6>(out, r[6], pend);
}

__device__ __forceinline__ void encode_col(uint32_t c_lo, uint32_t c_hi, uint32_t m_lo, uint32_t m_hi, uint32_t pend,
                                           uint32_t (&r)[7]) {
  uint32_t ty, co, st;
  encode4(c_lo, m_lo, ty, co, st);
  r[0] = prmt(ty, co, 0x5140);  // t0 c0 t1 c1
  r[1] = prmt(ty, co, 0x7362);  // t2 c2 t3 c3
  r[2] = st;
  encode4(c_hi, m_hi, ty, co, st);
  r[3] = prmt(ty, co, 0x5140);
  r[4] = prmt(ty, co, 0x7362);
  r[5] = st;
  r[6] = pend;
}

// View column vi (lateral offset vi-3) of one env as 7 cell bytes (byte vj
// = distance 6-vj from the agent) in clo (vj 0..3) / chi (vj 4..6), for
// grids up to 8x8: `lines` are this env's 8 SMEM lines (stride TILE), its grid
// rows when dir is even, its columns when dir is odd; one 64-bit load and two
// byte permutes per column.
//  dir 0: row    ay+vi-3, x = ax+6-vj     dir 1: column ax+3-vi, y = ay+6-vj
//  dir 2: row    ay+3-vi, x = ax-6+vj     dir 3: column ax+vi-3, y = ay-6+vj
// (P6 pins this closed form).  Positions outside the grid read arbitrary
// bytes: behind the closed wall border they can never become visible (R#12).
__device__ __forceinline__ void view_columns_narrow(const uint64_t* lines, int ax, int ay, int dir, uint32_t (&clo)[7],
                                                    uint32_t (&chi)[7]) {
  const int base = dir == 0 ? ay - 3 : dir == 1 ? ax + 3 : dir == 2 ? ay + 3 : ax - 3;
  const int sgn = (dir == 0 || dir == 3) ? 1 : -1;
  const int s = (dir == 0 ? ax : dir == 1 ? ay : dir == 2 ? ax - 6 : ay - 6) & 7;
  const bool rev = dir <= 1;
  const uint32_t s4 = (uint32_t)s * 0x1111u;
  // byte selectors: cell vj of the column = line byte (s + vj) or (s + 6 - vj), mod 8
  const uint32_t sel_lo = (s4 + (rev ? 0x3456u : 0x3210u)) & 0x7777u;
  const uint32_t sel_hi = (s4 + (rev ? 0x0012u : 0x7654u)) & 0x7777u;
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) {
    const uint64_t line = lines[((base + sgn * vi) & 7) * TILE];
    const uint32_t lo = (uint32_t)line, hi = (uint32_t)(line >> 32);
    clo[vi] = prmt(lo, hi, sel_lo);
    chi[vi] = prmt(lo, hi, sel_hi);
  }
}

// The same for grids wider than 8 (RW >= 2 u64 planes per row, row f2): row
// indices are clamped into the grid and word indices left of a row to word
// 0, so every load stays inside this env's planes (or, past the last row's
// last plane, in the SMEM that follows them); out-of-grid positions read
// arbitrary bytes (R#12).
template <int RW, int H>
__device__ __forceinline__ void view_columns_big(const uint64_t* rows, int ax, int ay, int dir, uint32_t (&clo)[7],
                                                 uint32_t (&chi)[7]) {
  const int base = dir == 0 ? ay - 3 : dir == 1 ? ax + 3 : dir == 2 ? ay + 3 : ax - 3;
  const int sgn = (dir == 0 || dir == 3) ? 1 : -1;
  const int s = dir == 0 ? ax : dir == 1 ? ay : dir == 2 ? ax - 6 : ay - 6;  // first position of the window
  const bool rev = dir <= 1;
  const uint8_t* rb = reinterpret_cast<const uint8_t*>(rows);  // plane p of this env at rb + p * TILE * 8
  constexpr int ROW_BYTES = RW * TILE * 8, PLANE_BYTES = TILE * 8;
  auto clamp_y = [](int y) { return y < 0 ? 0 : y > H - 1 ? H - 1 : y; };
  if ((dir & 1) == 0) {
    // the 7-byte window of a row from its 32-bit words q-2 .. q (virtual byte
    // offset s + 8 >= 2, so word indices are those of the row shifted by 2);
    // words left of the row only hold out-of-grid bytes: read word 0 instead
    const int sv = s + 8, q = sv >> 2, r = 8 * (sv & 3);
    auto woff = [](int k) { return (k >> 1) * PLANE_BYTES + (k & 1) * 4; };
    const int o0 = woff(q - 2 < 0 ? 0 : q - 2), o1 = woff(q - 1 < 0 ? 0 : q - 1), o2 = woff(q);
#pragma unroll
    for (int vi = 0; vi < 7; ++vi) {
      const uint8_t* rp = rb + clamp_y(base + sgn * vi) * ROW_BYTES;
      const uint32_t w0 = *reinterpret_cast<const uint32_t*>(rp + o0);
      const uint32_t w1 = *reinterpret_cast<const uint32_t*>(rp + o1);
      const uint32_t w2 = *reinterpret_cast<const uint32_t*>(rp + o2);
      const uint32_t f_lo = __funnelshift_r(w0, w1, r), f_hi = __funnelshift_r(w1, w2, r);
      clo[vi] = rev ? prmt(f_lo, f_hi, 0x3456u) : f_lo;
      chi[vi] = rev ? prmt(f_lo, f_hi, 0x0012u) : f_hi;
    }
  } else {
    // byte x of rows s .. s+6: the clamped row offsets are shared by the 7 columns
    int roff[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) roff[k] = clamp_y(s + k) * ROW_BYTES;
#pragma unroll
    for (int vi = 0; vi < 7; ++vi) {
      int x = base + sgn * vi;
      x = x < 0 ? 0 : x > 8 * RW - 1 ? 8 * RW - 1 : x;
      const uint8_t* cp = rb + (x >> 3) * PLANE_BYTES + ((x >> 2) & 1) * 4;
      const uint32_t xb = (uint32_t)(x & 3), pair = ((4u + xb) << 4) | xb;
      uint32_t w[7];
#pragma unroll
      for (int k = 0; k < 7; ++k) w[k] = *reinterpret_cast<const uint32_t*>(cp + roff[k]);
      const uint32_t p01 = prmt(w[0], w[1], pair), p23 = prmt(w[2], w[3], pair);
      const uint32_t p45 = prmt(w[4], w[5], pair), p6 = prmt(w[6], w[6], pair);
      const uint32_t f_lo = prmt(p01, p23, 0x5410u), f_hi = prmt(p45, p6, 0x5410u);  // cells y = s .. s+6
      clo[vi] = rev ? prmt(f_lo, f_hi, 0x3456u) : f_lo;
      chi[vi] = rev ? prmt(f_lo, f_hi, 0x0012u) : f_hi;
    }
  }
}

// Out-of-grid view cells as walls ([MG] gen_obs_grid's slice), for grids
// whose edge is not a closed wall border (GoToDoor, R#37).  Cell vj of
// column vi lies at lateral offset vi-3 and distance 6-vj from the agent.
template <int H, int W>
__device__ __forceinline__ void view_oob_walls(int ax, int ay, int dir, uint32_t (&clo)[7], uint32_t (&chi)[7]) {
  const int fx = dir == 0 ? 1 : dir == 2 ? -1 : 0, fy = dir == 1 ? 1 : dir == 3 ? -1 : 0;  // forward
  const int lx = -fy, ly = fx;                                                                // lateral +1
  uint32_t mlo = 0, mhi = 0;  // bytes along a column that leave the grid (forward component)
#pragma unroll
  for (int vj = 0; vj < 7; ++vj) {
    const int x = ax + (6 - vj) * fx, y = ay + (6 - vj) * fy;
    const bool out = fx ? (unsigned)x >= (unsigned)W : (unsigned)y >= (unsigned)H;
    if (vj < 4) mlo |= out ? 0xFFu << (8 * vj) : 0u;
    else mhi |= out ? 0xFFu << (8 * (vj - 4)) : 0u;
  }
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) {
    const int x = ax + (vi - 3) * lx, y = ay + (vi - 3) * ly;
    const bool out = lx ? (unsigned)x >= (unsigned)W : (unsigned)y >= (unsigned)H;
    const uint32_t m_lo = out ? 0xFFFFFFFFu : mlo, m_hi = out ? 0xFFFFFFFFu : mhi;
    clo[vi] = (clo[vi] & ~m_lo) | (0x01010101u * CELL_WALL & m_lo);
    chi[vi] = (chi[vi] & ~m_hi) | (0x01010101u * CELL_WALL & m_hi);
  }
}

// process_vis of the 7x7 view (byte vj of vis_lo / vis_hi has bit vi set iff
// view cell (vi, vj) is visible; bit 7 of each byte is garbage — the callers
// only ever move bit vi, vi <= 6, to a sign position).
// process_vis from the opacity rows: byte vj of op_lo (vj 0..3) / op_hi
// (vj 4..6) has bit vi set iff view cell (vi, vj) is opaque.
__device__ __forceinline__ void visibility_closure(uint32_t op_lo, uint32_t op_hi, uint32_t& vis_lo,
                                                   uint32_t& vis_hi) {
  // transparency rows and their 7-bit reversals (bit vi -> bit 6-vi)
  const uint32_t t_lo = ~op_lo & 0x7F7F7F7Fu, t_hi = ~op_hi & 0x7F7F7F7Fu;
  const uint32_t tr_lo = (prmt(__brev(t_lo), 0u, 0x0123u) >> 1) & 0x7F7F7F7Fu;
  const uint32_t tr_hi = (prmt(__brev(t_hi), 0u, 0x0123u) >> 1) & 0x7F7F7F7Fu;
  // rows vj = 6 .. 0 ([MG] process_vis order): V = R(S) | L(S), computed as
  // one carry chain on X = S | rev(S) << 8 over T2 = T | rev(T) << 8 (bit 7 = 0
  // stops the carry between the halves).  The seed stays in that doubled form
  // from row to row: dilation commutes with the reversal, so the next row's X
  // is the dilated (V | rev(V) << 8) & T2, masked back to bits 0-6 / 8-14.
  vis_lo = 0;
  vis_hi = 0;
  uint32_t x = (1u << 3) | (1u << 11);  // S = {vi = 3}, rev(S) = S
#pragma unroll
  for (int j = 6; j >= 0; --j) {
    const uint32_t tw = j < 4 ? t_lo : t_hi, trw = j < 4 ? tr_lo : tr_hi;
    const uint32_t b = (uint32_t)(j & 3);
    // t2 = T | rev(T) << 8 (bits 7 and 15 zero: carry stoppers; bytes 2-3
    // zero: selector 8 replicates the sign of byte 0 of tw, which is 0)
    const uint32_t t2 = prmt(tw, trw, 0x8800u | ((4u + b) << 4) | b);
    // x may carry garbage in bits 7 and 15: t2 masks it out of the carry
    // chains, and it only ever reaches bits 7 / 15 of v2 and w
    const uint32_t sum = t2 + (t2 & x);
    const uint32_t v2 = x | (sum ^ (t2 & ~x));  // R(S) | rev(L(S)) << 8 (carry chains)
    // V | rev(V) << 8 in bits 0-6 / 8-14 (bits 7 and 15: garbage)
    const uint32_t w = v2 | (__brev(v2) >> 17);
    const uint32_t av = w & t2;
    x = av | (av << 1) | (av >> 1);
    // byte 0 of w into byte j of the row masks
    const uint32_t sel = (0x3210u & ~(0xFu << (4 * b))) | (4u << (4 * b));
    if (j < 4) vis_lo = prmt(vis_lo, w, sel);
    else vis_hi = prmt(vis_hi, w, sel);
  }
}

__device__ __forceinline__ void view_visibility(const uint32_t (&clo)[7], const uint32_t (&chi)[7], uint32_t& vis_lo,
                                                uint32_t& vis_hi) {
  // opacity rows: byte vj of op has bit vi set iff cell (vi, vj) is opaque
  uint32_t op_lo = 0, op_hi = 0;
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) {
    op_lo |= (clo[vi] >> (7 - vi)) & (0x01010101u << vi);
    op_hi |= (chi[vi] >> (7 - vi)) & (0x01010101u << vi);
  }
  visibility_closure(op_lo, op_hi, vis_lo, vis_hi);
}

// Everything after the view columns and the visibility (view_visibility):
// encode, emission.
// out: word-aligned SMEM address at or before this env's record, whose first
// byte is at misalignment M (warp-uniform, 0..3).  All 7 columns are encoded
// first; only the emission is specialised on M (one warp-uniform switch), so
// the four variants share the rest of the code.
__device__ __forceinline__ void observe_cols(uint32_t (&clo)[7], uint32_t (&chi)[7], uint32_t carry, uint32_t* out,
                                             int M, uint32_t vis_lo, uint32_t vis_hi) {
  // the agent sees what it carries (R#13): view cell (3, 6), always visible
  chi[3] = prmt(chi[3], carry, 0x3410u);
  uint32_t r[7][7];
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) {
    const uint32_t m_lo = prmt(vis_lo * (1u << (7 - vi)), 0u, 0xBA98u);  // multiply: FMA pipe
    const uint32_t m_hi = prmt(vis_hi * (1u << (7 - vi)), 0u, 0xBA98u);
    encode_col(clo[vi], chi[vi], m_lo, m_hi, 0u, r[vi]);
  }
  switch (M) {  // one warp-uniform dispatch for the whole record
    case 0: emit_record<0>(out, r); break;
    case 1: emit_record<1>(out, r); break;
    case 2: emit_record<2>(out, r); break;
    default: emit_record<3>(out, r); break;
  }
}

// ---------------------------------------------------------------- one column
// The small-batch kernel (navix_step_wide) splits one env's observation over
// lanes: lane vi builds view column vi only.  Grids up to 8 wide; `rows` are
// the env's 8 SMEM row lines (stride TILE).  Even directions read one world
// row (as view_columns_narrow); odd ones gather the world column byte by byte
// (no in-place transpose: the rows are shared by the env's lanes).
__device__ __forceinline__ void view_column_narrow(const uint64_t* rows, int ax, int ay, int dir, int vi,
                                                   uint32_t& clo, uint32_t& chi) {
  const int base = dir == 0 ? ay - 3 : dir == 1 ? ax + 3 : dir == 2 ? ay + 3 : ax - 3;
  const int sgn = (dir == 0 || dir == 3) ? 1 : -1;
  const int s = (dir == 0 ? ax : dir == 1 ? ay : dir == 2 ? ax - 6 : ay - 6) & 7;
  const bool rev = dir <= 1;
  const uint32_t s4 = (uint32_t)s * 0x1111u;
  const uint32_t sel_lo = (s4 + (rev ? 0x3456u : 0x3210u)) & 0x7777u;
  const uint32_t sel_hi = (s4 + (rev ? 0x0012u : 0x7654u)) & 0x7777u;
  const int li = (base + sgn * vi) & 7;
  uint32_t lo, hi;
  if ((dir & 1) == 0) {
    const uint64_t line = rows[li * TILE];
    lo = (uint32_t)line;
    hi = (uint32_t)(line >> 32);
  } else {  // world column li: byte y = cell (li, y)
    const uint8_t* b = reinterpret_cast<const uint8_t*>(rows) + li;
    constexpr int R = TILE * 8;  // bytes between row lines
    lo = prmt(prmt(b[0], b[R], 0x0040u), prmt(b[2 * R], b[3 * R], 0x0040u), 0x5410u);
    hi = prmt(prmt(b[4 * R], b[5 * R], 0x0040u), prmt(b[6 * R], b[7 * R], 0x0040u), 0x5410u);
  }
  clo = prmt(lo, hi, sel_lo);
  chi = prmt(lo, hi, sel_hi);
}

// The 21 record bytes of one encoded column (encode_col's registers r[0..5])
// in stream order (t c s per cell vj), stored byte by byte at dst.
__device__ __forceinline__ void store_column_bytes(uint8_t* dst, const uint32_t (&r)[7]) {
  // r0 = t0 c0 t1 c1, r1 = t2 c2 t3 c3, r2 = s0 s1 s2 s3, r3 = t4 c4 t5 c5, r4 = t6 c6 . ., r5 = s4 s5 s6 .
  const uint32_t w0 = prmt(r[0], r[2], 0x2410u);                      // t0 c0 s0 t1
  const uint32_t w1 = prmt(prmt(r[0], r[2], 0x0053u), r[1], 0x5410u);  // c1 s1 t2 c2
  const uint32_t w2 = prmt(r[1], r[2], 0x7326u);                      // s2 t3 c3 s3
  const uint32_t w3 = prmt(r[3], r[5], 0x2410u);                      // t4 c4 s4 t5
  const uint32_t w4 = prmt(prmt(r[3], r[5], 0x0053u), r[4], 0x5410u);  // c5 s5 t6 c6
  const uint32_t w[5] = {w0, w1, w2, w3, w4};
#pragma unroll
  for (int k = 0; k < 20; ++k) dst[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
  dst[20] = (uint8_t)(r[5] >> 16);                                    // s6
}

// ---------------------------------------------------------------- categorical
// categorical_first_person (Table 5, R#41): the 49-byte record of view
// cell types [vi][vj].  Stream byte i of the record is type byte i % 7 of
// column i / 7; word K of the word-aligned output gathers its <= 4 bytes from
// at most two type registers (t[2 vi] = vj 0..3, t[2 vi + 1] = vj 4..6), so
// one byte permute per word with a compile-time selector.
struct CatPlan {
  int p0, p1;      // valid byte range of the word (p0 > p1: nothing to store)
  int s0, s1;      // source registers
  uint32_t sel;
};
__host__ __device__ constexpr CatPlan cat_plan(int M, int K) {
  CatPlan P{4, -1, 0, 0, 0u};
  int src[2] = {-1, -1};
  uint32_t sel = 0;
  for (int p = 0; p < 4; ++p) {
    const int i = 4 * K + p - M;
    if (i < 0 || i > 48) continue;
    if (P.p0 > p) P.p0 = p;
    P.p1 = p;
    const int col = i / 7, vj = i % 7;
    const int reg = 2 * col + (vj >= 4 ? 1 : 0), byt = vj & 3;
    int slot = src[0] == reg ? 0 : src[1] == reg ? 1 : src[0] < 0 ? 0 : 1;
    src[slot] = reg;
    sel |= (uint32_t)(4 * slot + byt) << (4 * p);
  }
  P.s0 = src[0] < 0 ? 0 : src[0];
  P.s1 = src[1] < 0 ? P.s0 : src[1];
  P.sel = sel;
  return P;
}
template <int M, int K>
__device__ __forceinline__ void emit_cat_word(uint32_t* out, const uint32_t (&t)[14]) {
  constexpr CatPlan P = cat_plan(M, K);
  if constexpr (P.p0 <= P.p1) {
    const uint32_t v = prmt(t[P.s0], t[P.s1], P.sel);
    if constexpr (P.p0 == 0 && P.p1 == 3) out[K] = v;
    else sts_bytes(out + K, v, P.p0, P.p1);
  }
}
template <int M>
__device__ __forceinline__ void emit_cat_record(uint32_t* out, const uint32_t (&t)[14]) {
  emit_cat_word<M, 0>(out, t);  emit_cat_word<M, 1>(out, t);  emit_cat_word<M, 2>(out, t);
  emit_cat_word<M, 3>(out, t);  emit_cat_word<M, 4>(out, t);  emit_cat_word<M, 5>(out, t);
  emit_cat_word<M, 6>(out, t);  emit_cat_word<M, 7>(out, t);  emit_cat_word<M, 8>(out, t);
  emit_cat_word<M, 9>(out, t);  emit_cat_word<M, 10>(out, t); emit_cat_word<M, 11>(out, t);
  emit_cat_word<M, 12>(out, t);
}
// type-only SWAR encode (encode4 without colour and state)
__device__ __forceinline__ uint32_t encode4_type(uint32_t w, uint32_t m) {
  const uint32_t E = w & m & 0x0F0F0F0Fu;
  uint32_t D;
  asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(D) : "r"(E + 0x75757575u));
  return (E & ~D) | (D & 0x04040404u);
}
__device__ __forceinline__ void observe_cols_cat(uint32_t (&clo)[7], uint32_t (&chi)[7], uint32_t carry,
                                                 uint32_t* out, int M, uint32_t vis_lo, uint32_t vis_hi) {
  chi[3] = prmt(chi[3], carry, 0x3410u);  // the agent sees what it carries (R#13)
  uint32_t t[14];
#pragma unroll
  for (int vi = 0; vi < 7; ++vi) {
    const uint32_t m_lo = prmt(vis_lo * (1u << (7 - vi)), 0u, 0xBA98u);
    const uint32_t m_hi = prmt(vis_hi * (1u << (7 - vi)), 0u, 0xBA98u);
    t[2 * vi] = encode4_type(clo[vi], m_lo);
    t[2 * vi + 1] = encode4_type(chi[vi], m_hi);
  }
  switch (M) {
    case 0: emit_cat_record<0>(out, t); break;
    case 1: emit_cat_record<1>(out, t); break;
    case 2: emit_cat_record<2>(out, t); break;
    default: emit_cat_record<3>(out, t); break;
  }
}

}  // namespace navix
