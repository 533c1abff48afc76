// step_kernel.cuh — the fused batched MiniGrid step for sm_100a (kernel templates;
// instantiated per family group in inst_*.cu, dispatched in dispatch.cu).
//
// One thread owns one environment; one CTA owns a tile of TILE = 128 envs.
// Per env and step:
//   a1 stage      TMA bulk copies (cp.async.bulk + mbarrier) of the tile's grid
//                 row planes, agent records and actions into SMEM; the
//                 persistent kernel prefetches the next tile while it computes
//   a2 autoreset  if the previous step ended: episode += 1, Philox level
//                 generation into the SMEM rows (levelgen.cuh), first obs
//   a3 transition Dynamic-Obstacles balls (Table 3, App. A)
//   a4 intervene  left/right/forward/pickup/drop/toggle/done,
//                 branch-free
//   a5 reward     Eq. (1) P:216 / P:223 (R#1-R#3), events -> terminated,
//                 step_count >= T -> truncated (R#17); Table 6/7 selection and
//                 costs (R#31, R#42)
//   a6 observe    symbolic_first_person (Table 5) or its categorical
//                 form (R#41): the 7 view columns are 7 world lines shifted
//                 and byte-reversed; MiniGrid's process_vis as 7-bit row
//                 closures computed with one integer add each (carry =
//                 propagation); SWAR encode of 4 cells per 32-bit word; the
//                 record assembled in registers at its final byte alignment
//   a7 store      obs staged in SMEM, written by ONE cp.async.bulk per tile;
//                 reward/flags/agent records coalesced; a modified grid plane
//                 written back only when an action changed it; episode
//                 statistics warp-reduced into striped int64 counters.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "layout.h"
#include "levelgen.cuh"
#include "obs.cuh"
#include "philox.cuh"

#ifndef NAVIX_KC_WARP_MAX
#define NAVIX_KC_WARP_MAX 4
#endif

namespace navix {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mbarrier + TMA bulk copy (global -> shared) primitives
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 1000000;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}" ::"r"(mbar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(mbar)
               : "memory");
}

// 8x8 byte transpose of one env's lines in place: rows (byte x of line y) ->
// columns (byte y of line x), 32 byte permutes.
__device__ __forceinline__ void transpose4x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t& o0,
                                             uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  o0 = __byte_perm(t0, t1, 0x5410);
  o1 = __byte_perm(t0, t1, 0x7632);
  o2 = __byte_perm(t2, t3, 0x5410);
  o3 = __byte_perm(t2, t3, 0x7632);
}

// (src == dst: in place; the rollout transposes into scratch lines, keeping
// the rows for the next step)
__device__ __forceinline__ void transpose_lines(const uint64_t* src, uint64_t* lines) {
  uint32_t lo[8], hi[8];
#pragma unroll
  for (int y = 0; y < 8; ++y) {
    const uint64_t r = src[y * TILE];
    lo[y] = (uint32_t)r;
    hi[y] = (uint32_t)(r >> 32);
  }
  uint32_t a[4], b[4], c[4], d[4];
  transpose4x4(lo[0], lo[1], lo[2], lo[3], a[0], a[1], a[2], a[3]);  // x 0..3, y 0..3
  transpose4x4(lo[4], lo[5], lo[6], lo[7], b[0], b[1], b[2], b[3]);  // x 0..3, y 4..7
  transpose4x4(hi[0], hi[1], hi[2], hi[3], c[0], c[1], c[2], c[3]);  // x 4..7, y 0..3
  transpose4x4(hi[4], hi[5], hi[6], hi[7], d[0], d[1], d[2], d[3]);  // x 4..7, y 4..7
#pragma unroll
  for (int x = 0; x < 8; ++x)
    lines[x * TILE] = x < 4 ? ((uint64_t)b[x] << 32) | a[x] : ((uint64_t)d[x - 4] << 32) | c[x - 4];
}

static __device__ __noinline__ float success_reward(int mode, uint32_t sc, uint32_t T) {
  if (mode == 1) return 1.0f;
  // R#2: binary64, [MG] order, no contraction, one rounding to binary32
  const double q = __ddiv_rn((double)sc, (double)T);
  const double p = __dmul_rn(0.9, q);
  return __double2float_rn(__dsub_rn(1.0, p));
}

// ------------------------------------------------------------------ tile body
// Lane <-> env mapping inside a tile: thread tid = 32*w + l (warp w, lane l)
// owns tile-local env le = 4*l + w.  All state arrays are indexed by the
// "slot" tid, so every warp access to them is contiguous; caller arrays
// (actions, obs, reward, flags) are indexed by the env.  A warp's envs then
// share le mod 4, so their 147-byte records start at the same byte
// misalignment M = 147*le mod 4 = 3w mod 4 and the record emission is
// specialised per warp at compile time (no per-lane shifts, and the
// per-lane SMEM word stride 147 is odd: bank-conflict free).

// One tile's input buffers in SMEM (filled by TMA bulk copies).
template <int FAM, int NPL>
struct TileSmem {
  uint64_t rows[NPL][TILE];                          // grid row planes; later this env's view lines
  uint64_t agent[TILE];                              // agent records
  uint64_t balls[FAM == FAM_DYNOBS ? TILE : 2];      // DynObs ball positions
  uint32_t episode[FAM == FAM_DYNOBS ? TILE : 4];    // DynObs episode counters
  uint8_t act[TILE];                                 // actions (env order)
};

// Thread 0: bulk-copy tile `tile`'s inputs into `b`, completing on `mbar`.
// Returns whether the actions came along (full tile, 16-B aligned base).
template <int FAM, int HP, int MODE, int NPL>
__device__ __forceinline__ bool issue_tile_loads(const KernelArgs& a, int64_t tile, TileSmem<FAM, NPL>& b,
                                                 uint32_t mbar) {
  // HP = grid planes per env (H rows x RW u64)
  const int64_t tile0 = tile * TILE;
  const bool act_bulk = MODE == MODE_STEP && a.bulk_act && tile0 + TILE <= a.n;
  const uint32_t bytes = HP * TILE * 8 + TILE * 8 + (act_bulk ? TILE : 0) +
                         (FAM == FAM_DYNOBS ? (MODE == MODE_STEP ? 12 : 8) * TILE : 0);
  mbar_expect_tx(mbar, bytes);
  bulk_g2s(&b.rows[0][0], a.grid + tile0 * HP, HP * TILE * 8, mbar);
  bulk_g2s(b.agent, a.agent + tile0, TILE * 8, mbar);
  if (act_bulk) bulk_g2s(b.act, a.actions + tile0, TILE, mbar);
  if (FAM == FAM_DYNOBS) {
    bulk_g2s(b.balls, a.balls + tile0, TILE * 8, mbar);
    if (MODE == MODE_STEP) bulk_g2s(b.episode, a.episode + tile0, TILE * 4, mbar);
  }
  return act_bulk;
}

// Everything a tile does once its inputs are in SMEM (MODE != RESET) or
// without inputs (RESET): a2-a7 for this thread's env, the obs bulk store
// issued by thread 0 (the caller waits for it before reusing s_obs).
// Per-thread results of a tile, written out by tile_store().
struct EnvResult {
  float reward;
  bool valid, regen, term, trunc, dirty;
  bool tvalid;  // rollout: the scratch lines hold the transpose of the current rows
  uint64_t nrec, balls;
  uint32_t episode;
  uint32_t st[8];
};

// The state a padding slot (env index >= n in the last tile) is stepped with:
// its HBM record is never written (caller-owned state buffers hold whatever
// was there), so it is replaced by a legal pose — (1, 1) east, nothing
// carried, no flags — and no balls; its results are never stored.
constexpr uint64_t PADDING_AGENT_RECORD = 0x0000000001000101ull;

// One env's inputs for a step (decoded from the staged tile, or carried in
// registers across the steps of a rollout).
struct EnvIn {
  uint64_t rec;      // agent record
  uint32_t act;      // action
  uint64_t balls;    // DynObs ball positions (byte b = ball_code(W, x, y), layout.h)
  uint32_t episode;  // episode counter
  bool episode_known;  // else read from HBM when an auto-reset needs it
  bool tvalid;         // rollout: the scratch lines hold the transpose of these rows
  bool rows_persist;   // rollout: the SMEM rows are last step's (not reloaded from HBM)
};

template <int FAM, int MODE, int NPL>
__device__ __forceinline__ EnvIn decode_staged(const KernelArgs& a, int64_t tile, const TileSmem<FAM, NPL>& b) {
  const int tid = threadIdx.x, le = 4 * (tid & 31) + (tid >> 5);
  const int64_t tile0 = tile * TILE, e = tile0 + le;
  EnvIn in{0, 0, 0, 0, false};
  if (MODE != MODE_RESET) {
    in.rec = b.agent[tid];
    if (MODE == MODE_STEP && e < a.n) {
      const bool act_bulk = a.bulk_act && tile0 + TILE <= a.n;
      in.act = act_bulk ? b.act[le] : a.actions[e];
    }
    if (FAM == FAM_DYNOBS) {
      in.balls = b.balls[tid];
      if (MODE == MODE_STEP) {
        in.episode = b.episode[tid];
        in.episode_known = true;
      }
    }
    if (e >= a.n) {  // padding slot of the last tile: never written, may hold anything
      in.rec = PADDING_AGENT_RECORD;
      in.balls = 0;
    }
  }
  return in;
}

// The per-CTA reset-queue counter of the Dynamic-Obstacles / GoToDoor step
// (tile_compute).  Zero on entry: every kernel that steps those families
// zeroes it before its first CTA barrier (init_reset_queue_counter), and
// tile_compute zeroes it again once the queue is consumed.
__device__ __forceinline__ int& reset_queue_counter() {
  __shared__ int s_qn;
  return s_qn;
}
// its slot list: written before the queue's first barrier, so it cannot live
// in the tile's action staging (slower warps may still be decoding it)
__device__ __forceinline__ uint8_t* reset_queue_slots() {
  __shared__ uint8_t s_qslot[TILE];
  return s_qslot;
}
template <int FAM>
__device__ __forceinline__ void init_reset_queue_counter() {
  if (FAM == FAM_DYNOBS || FAM == FAM_GOTODOOR)
    if (threadIdx.x == 0) reset_queue_counter() = 0;
}

// ------------------------------------------------------------------ visibility table
// Static-layout families (STATIC_LAYOUT: Dynamic-Obstacles, Empty,
// Empty-Random, DistShift): the layout is the family's template and balls are
// see-through, so MiniGrid's process_vis mask is a function of the agent pose
// alone.  Per pose ((ay-1)(W-2) + ax-1) * 4 + dir: (vis_lo, vis_hi) as
// view_visibility returns them, built by obs_table_kernel with that very
// function on the template grid.  One table per device (a __device__
// variable), built at handle creation (navix_create_shard).
// DoorKey (LAYOUT_KEYED_VIS): one such table per layout key (split, door_y,
// door open), key-major.
template <int FAM, int H, int W>
constexpr int vis_table_layouts() {
  return LAYOUT_KEYED_VIS<FAM, W> ? (W - 4) * (W - 3) * 2 : 1;
}
template <int FAM, int H, int W>
__device__ uint2 g_vis_table[vis_table_layouts<FAM, H, W>() * (W - 2) * (H - 2) * 4];

template <int FAM, int H, int W>
__device__ __forceinline__ const uint2* obs_table_entry(int ax, int ay, int dir, int layout = 0) {
  return g_vis_table<FAM, H, W> + (layout * (W - 2) * (H - 2) + (ay - 1) * (W - 2) + (ax - 1)) * 4 + dir;
}

template <int FAM, int H, int W>
__global__ void __launch_bounds__(TILE) obs_table_kernel() {
  using C = Cfg<FAM, H, W>;
  // + 2 zero planes: view_columns_big may read up to two planes past the last
  // row (the step kernels have other SMEM there; never visible, R#12)
  __shared__ uint64_t rows_s[C::NPL + 2][TILE];
  const int tid = threadIdx.x;
  const int entry = blockIdx.x * TILE + tid;
  constexpr int NPOSE = (W - 2) * (H - 2) * 4;
  if (entry >= vis_table_layouts<FAM, H, W>() * NPOSE) return;
  const int pose = entry % NPOSE, layout = entry / NPOSE;
  const int dir = pose & 3, cell = pose >> 2;
  const int ax = 1 + cell % (W - 2), ay = 1 + cell / (W - 2);
  uint64_t* rows = &rows_s[0][tid];
  if constexpr (LAYOUT_KEYED_VIS<FAM, W>) {
    // border walls, the wall column, its door (locked or open)
    const int split = 2 + (layout >> 1) / (W - 3), door_y = 1 + (layout >> 1) % (W - 3);
    const bool open = layout & 1;
    RowViewT<1> g{rows};
#pragma unroll
    for (int y = 0; y < 8; ++y) rows[y * TILE] = 0ull;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const bool wall = x == 0 || y == 0 || x == W - 1 || y == H - 1 || x == split;
        g.set(x, y, wall ? CELL_WALL : CELL_EMPTY);
      }
    g.set(split, door_y, open ? make_cell(K_DOOR_OPEN, COL_YELLOW) : make_cell(K_DOOR_LOCKED, COL_YELLOW));
  } else {
#pragma unroll
    for (int p = 0; p < C::NPL + 2; ++p) rows[p * TILE] = p < H * C::RW ? template_plane<FAM, H, W>(p) : 0ull;
  }
  uint32_t clo[7], chi[7];
  if constexpr (C::RW == 1) {
    if (dir & 1) transpose_lines(rows, rows);
    view_columns_narrow(rows, ax, ay, dir, clo, chi);
  } else {
    view_columns_big<C::RW, H>(rows, ax, ay, dir, clo, chi);
  }
  uint32_t vis_lo, vis_hi;
  view_visibility(clo, chi, vis_lo, vis_hi);
  g_vis_table<FAM, H, W>[entry] = make_uint2(vis_lo, vis_hi);
}

// a1-a6 for this thread's env: compute, then write its obs record into s_obs
// (after before_emit() has made sure s_obs is free).  rows: this env's 8 SMEM
// row lines (stride TILE); scratch: 8 more lines for the column view of odd
// directions, or nullptr to transpose the rows in place (then the rows are
// written back to HBM first if the grid changed, and are lost).
//
// WIDE (navix_step_wide, small batches): WIDE_LANES consecutive lanes share
// one env, tile-local env `wide_le`, and all compute its step redundantly on
// the same inputs (their SMEM writes are identical); there is no CTA queue or
// warp-cooperative generator, the grid write-back is split over the lanes,
// and the function returns before the observation, which the lanes split by
// view column (navix_step_wide).
constexpr int WIDE_LANES = 8;
template <int FAM, int H, int W, int MODE, int OBSK, class BeforeEmit, bool WIDE = false>
__device__ __forceinline__ EnvResult tile_compute(const KernelArgs& a, int64_t tile, uint64_t* rows, uint64_t* scratch,
                                                  const EnvIn& in, uint8_t* s_obs, BeforeEmit before_emit,
                                                  int wide_le = 0) {
  using C = Cfg<FAM, H, W>;
  // state slot and env of this thread within the tile (layout.h: slot 32 w + l <-> env 4 l + w)
  const int tid = WIDE ? slot_of_env(wide_le) : (int)threadIdx.x;
  const int warp = tid >> 5, lane = WIDE ? (int)(threadIdx.x & 31) : tid & 31;
  const int le = WIDE ? wide_le : 4 * lane + warp;
  const int64_t tile0 = tile * TILE;
  const int64_t slot = tile0 + tid;   // state index
  const int64_t e = tile0 + le;       // env index (caller arrays)
  const bool valid = e < a.n;
  const uint32_t genv = a.env_begin + (uint32_t)e;  // global env index: Philox counter word c0
  constexpr int RW = C::RW;
  RowViewT<RW> g{rows};

  // ---- a1: inputs
  uint8_t act = (uint8_t)in.act;
  const uint64_t rec = in.rec;
  uint64_t balls = in.balls;
  uint32_t episode = in.episode;
  int ax = (int)(rec & 0xFF), ay = (int)((rec >> 8) & 0xFF), dir = (int)((rec >> 16) & 3);
  uint8_t carry = (uint8_t)(rec >> 24);
  uint32_t sc = (uint32_t)((rec >> 32) & 0xFFFF);
  bool prev_done = (rec >> 48) & 1;
  // Dynamic-Obstacles: agent-record flag bit 1 = "this env's HBM grid already
  // holds the static template" (balls live outside it), so a reset need not
  // write the template back again
  // Static-layout families (STATIC_LAYOUT, levelgen.cuh: Dynamic-Obstacles,
  // Empty, Empty-Random, DistShift): agent-record flag bit 1 = "this env's
  // HBM grid holds the family's template", set by every generated level and
  // by imports of that layout, cleared by any change of a cell (pickup /
  // drop / toggle of imported objects); a reset need not write the template
  // back, and the visibility comes from the per-pose table
  bool grid_tmpl = STATIC_LAYOUT<FAM> && ((rec >> 49) & 1);
  // GoToDoor target door; DoorKey (split << 4) | door_y of its generated layout
  uint32_t target = (FAM == FAM_GOTODOOR || FAM == FAM_DOORKEY) ? (uint32_t)(rec >> 56) : 0u;
  // DoorKey: agent-record flag bit 2 = "the layout is a generated DoorKey
  // layout described by byte 7" (set by generation and by matching imports;
  // no action can change its opacity except the door's own toggle)
  // (LavaGap / lava Crossings, BORDER_OPACITY: the same flag says "the only
  // opaque cells are the border")
  constexpr bool KEYED_VIS = LAYOUT_KEYED_VIS<FAM, W> || BORDER_OPACITY<FAM>;
  bool layout_key = KEYED_VIS && ((rec >> 50) & 1);
  // GoToDoor: the same flag says "a generated room, no door opened since":
  // the room's walls and closed doors enclose the agent, so no cell outside
  // the room — and no position outside the grid — can become visible
  // (process_vis only spreads from visible see-through cells, all inside the
  // room), and the view needs no out-of-grid walls (R#37)
  bool room_closed = FAM == FAM_GOTODOOR && ((rec >> 50) & 1);

  float reward = 0.f;
  bool term = false, trunc = false, grid_dirty = false;
  int dirty_plane = -1;  // the one row plane an action modified; -1: all (a new level)
  uint32_t st_ep = 0, st_len = 0, st_succ = 0, st_succ_len = 0, st_lava = 0, st_coll = 0, st_trunc = 0,
           st_fail = 0;

  const bool regen = MODE == MODE_RESET || (MODE == MODE_STEP && prev_done);
  // Dynamic-Obstacles auto-resets ~10 % of its envs per step (GoToDoor ~30 %
  // under a random policy): left in place, nearly every warp would run the
  // level generator for a few lanes.  Their resetting envs are queued per CTA
  // instead and generated by the first threads (one warp for up to 32 of
  // them), each into its env's SMEM rows.
  // The queue now serves GoToDoor and the Dynamic-Obstacles-Random ids: the
  // fixed-start Dynamic-Obstacles ids generate in place without a generator
  // call (BITBOARD / UNIFIED_ROWS below; DynObs-16x16 174 -> 126.5 us per
  // 2^20-env step against the queue, which had itself taken it from 198).
  // (A warp-local queue — ballot, one generator pass per warp, no CTA barrier —
  // measured worse, DynObs-8x8 79 -> 91 us at 2^20: four passes per tile
  // instead of one, on an ALU-pipe-bound kernel.  GoToDoor's 4 Philox blocks
  // per level computed by the whole CTA ahead of the generator pass, through
  // s_obs: 67.7 -> 69.3 us at 2^20, an extra barrier for no shorter pass.)
  constexpr bool COMPACT = (FAM == FAM_DYNOBS || FAM == FAM_GOTODOOR) && MODE == MODE_STEP && !WIDE;
  constexpr bool KC_WARP = FAM == FAM_KEYCORRIDOR && MODE == MODE_STEP && !WIDE;
  constexpr int KC_WARP_MAX = NAVIX_KC_WARP_MAX;
  // Fixed-start Dynamic-Obstacles on grids up to 8 wide (BITBOARD below):
  // resetting lanes place their balls in the same bitboard loop that moves
  // the other lanes' balls, so they need neither the queue nor the generator
  constexpr bool BITBOARD = FAM == FAM_DYNOBS && RW == 1 && MODE == MODE_STEP;
  // Wider fixed-start Dynamic-Obstacles grids (16x16) generate in place too:
  // the resetting lanes place their balls by list index (below, no mask, no
  // queue), the other lanes move theirs on the SMEM rows (a3)
  constexpr bool UNIFIED_ROWS = FAM == FAM_DYNOBS && RW > 1 && MODE == MODE_STEP && !WIDE;
  const bool unified = (BITBOARD || UNIFIED_ROWS) && a.gen_param == 0;  // grid-uniform
  if (COMPACT && !unified) {
    // Agent record st of the staging this tile has consumed holds (episode |
    // generator output << 32) (each thread overwrites only the record it
    // decoded itself), DynObs ball word st the new balls; 132 B of static
    // SMEM for the counter and the slot list.  The counter is zero on entry
    // (by thread 0 before the kernel's first barrier, and below after its
    // last read), so filling the queue needs no barrier of its own.
    int& s_qn = reset_queue_counter();
    auto* const tb = reinterpret_cast<TileSmem<FAM, C::NPL>*>(rows - tid);
    uint8_t* const q_slot = reset_queue_slots();
    uint64_t* const q_rec = tb->agent;
    uint64_t* const q_balls = tb->balls;
    const unsigned rm = __ballot_sync(0xffffffffu, regen);
    int qbase = 0;
    if (lane == 0 && rm) qbase = atomicAdd(&s_qn, __popc(rm));  // one atomic per warp
    qbase = __shfl_sync(0xffffffffu, qbase, 0);
    if (regen) {
      q_slot[qbase + __popc(rm & ((1u << lane) - 1u))] = (uint8_t)tid;
      q_rec[tid] = (uint64_t)((in.episode_known ? episode : a.episode[slot]) + 1);
    }
    __syncthreads();
    const int nq = s_qn;
    for (int q = tid; q < nq; q += TILE) {
      const int st = q_slot[q];
      const uint32_t genv_t = a.env_begin + (uint32_t)(tile0 + env_of_slot(st));
      const uint32_t ep = (uint32_t)q_rec[st];
      const GenOut o = generate_level<FAM, H, W>(RowViewT<RW>{rows - tid + st}, genv_t, ep, a.key_lo, a.key_hi,
                                                 a.gen_param);
      if (FAM == FAM_DYNOBS) q_balls[st] = o.balls;
      const uint32_t out = (uint32_t)o.ax | ((uint32_t)o.ay << 8) | ((uint32_t)o.dir << 16) |
                           ((o.fail < 63u ? o.fail : 63u) << 18) | ((o.target & 0xFFu) << 24);
      q_rec[st] = (uint64_t)ep | ((uint64_t)out << 32);
    }
    __syncthreads();
    // every read of the counter happened before the barrier above; the next
    // tile's (or step's) atomics come after at least one more CTA barrier
    if (tid == 0) s_qn = 0;
    if (regen) {
      const uint64_t qr = q_rec[tid];
      const uint32_t o = (uint32_t)(qr >> 32);
      episode = (uint32_t)qr;
      if (FAM == FAM_GOTODOOR) {
        target = o >> 24;
        room_closed = true;
      } else {
        balls = q_balls[tid];
      }
      ax = (int)(o & 0xFF); ay = (int)((o >> 8) & 0xFF); dir = (int)((o >> 16) & 3);
      st_fail = (o >> 18) & 63u;
      carry = CELL_EMPTY;
      sc = 0;
      prev_done = false;
      grid_dirty = !grid_tmpl;
      grid_tmpl = STATIC_LAYOUT<FAM>;
    }
  } else if (KC_WARP || (regen && !unified)) {
    // ---- a2: next-step auto-reset (R#18) / reset(key)
    if (MODE == MODE_STEP && regen) {
      if (!in.episode_known) episode = a.episode[slot];
      episode += 1;
    }
    GenOut o;
    if constexpr (KC_WARP) {
      // KeyCorridor's connect_all loop (mean 25, tail > 150 iterations) made
      // one resetting lane the straggler of its tile and of the step.  When
      // few lanes of the warp reset, the whole warp generates each of their
      // levels in turn with 32 loop iterations per round; when many do (all
      // random-policy episodes truncate together at T), one lane per level.
      unsigned m = __ballot_sync(0xffffffffu, regen);
      if (__popc(m) > KC_WARP_MAX) {
        if (regen) o = generate_level<FAM, H, W>(g, genv, episode, a.key_lo, a.key_hi, a.gen_param);
      } else {
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t ep_l = __shfl_sync(0xffffffffu, episode, l);
          const uint32_t genv_l = __shfl_sync(0xffffffffu, genv, l);
          const GenOut ol = generate_level<FAM, H, W, true>(RowViewT<RW>{rows - lane + l}, genv_l, ep_l, a.key_lo,
                                                             a.key_hi, a.gen_param);
          if (lane == l) o = ol;
        }
      }
    } else {
      o = generate_level<FAM, H, W>(g, genv, episode, a.key_lo, a.key_hi, a.gen_param);
    }
    if (regen) {
      ax = o.ax; ay = o.ay; dir = o.dir;
      target = o.target;
      room_closed = FAM == FAM_GOTODOOR;
      layout_key = LAYOUT_KEYED_VIS<FAM, W> ||
                   (BORDER_OPACITY<FAM> && (FAM != FAM_CROSSING || (a.gen_param & CROSSING_LAVA)));
      balls = o.balls;
      st_fail = o.fail;
      carry = CELL_EMPTY;
      sc = 0;
      prev_done = false;
      grid_dirty = !grid_tmpl;
      grid_tmpl = STATIC_LAYOUT<FAM>;
    }
  }
  // Dynamic-Obstacles on grids up to 8 wide: the transition runs on 64-bit
  // bitboards (bit 8y + x) and the balls are overlaid into the SMEM rows once,
  // after they moved.  A warp whose envs all hold MiniGrid's static layout in
  // HBM (agent-record flag, set by every generated level and by imports of
  // that layout) takes the free cells from the compile-time template; a warp
  // with another imported layout builds them from its rows.  With a fixed
  // start (not -Random), the lanes whose env auto-resets run the SAME loop to
  // place their new level's balls (levelgen.cuh's DynObs generator: each ball
  // uniform over the template's empty cells minus the agent (1,1) and the
  // balls placed before it, draw b = word b of block (env, episode, 0, 0)):
  // no queue, no CTA barrier, no divergent generator call.
  auto overlay_balls = [&] {
#pragma unroll
    for (int bb = 0; bb < C::NOBST; ++bb) {
      const uint32_t p = (uint32_t)(balls >> (8 * bb)) & 0xFF;
      if (p) g.set(ball_x(W, p), ball_y(W, p), make_cell(K_BALL, COL_BLUE));
    }
  };
  bool not_clear_pre = false;  // DynObs: the front cell before the motion is not empty / goal
  if constexpr (BITBOARD) {
    const bool gen = unified && regen;  // this lane generates its next level here
    const uint64_t balls_before = balls;
    if (gen) {
      // a2 (R#18): episode e+1 of [MG] DynamicObstaclesEnv, agent (1,1) east
      episode = (in.episode_known ? episode : a.episode[slot]) + 1u;
      ax = 1; ay = 1; dir = 0;
      carry = CELL_EMPTY;
      sc = 0;
      prev_done = false;
      if (!grid_tmpl) {  // an imported layout: back to the template (SMEM now, HBM at write-back)
#pragma unroll
        for (int y = 0; y < H; ++y) rows[y * TILE] = template_plane<FAM, H, W>(y);
      }
      grid_dirty = !grid_tmpl;
      grid_tmpl = true;
      balls = 0;
    }
    const bool warp_tmpl = __all_sync(0xffffffffu, grid_tmpl);
    const bool move = !regen;
    if (move && act >= 3) act = 0;  // R#7
    if (move || gen) {
      // admissible cells: empty in the static layout, no ball, not the agent
      uint64_t freeb;
      if (warp_tmpl || gen) {
        freeb = template_free_cells<FAM, H, W>();
      } else {
        freeb = 0;
#pragma unroll
        for (int y = 0; y < H; ++y) {
          const uint64_t x = rows[y * TILE] ^ 0x0101010101010101ull;  // empty byte -> 0
          const uint64_t z = ~(((x & 0x7F7F7F7F7F7F7F7Full) + 0x7F7F7F7F7F7F7F7Full) | x | 0x7F7F7F7F7F7F7F7Full);
          freeb |= (((z >> 7) * 0x0102040810204080ull) >> 56) << (8 * y);  // bit x: byte x == 0
        }
      }
      // the ball byte is its bit index (ball_code); 0 = no ball clears bit 0,
      // the corner (0, 0), which is never free
#pragma unroll
      for (int bb = 0; bb < C::NOBST; ++bb) freeb &= ~(1ull << ((uint32_t)(balls >> (8 * bb)) & 0xFF));
      freeb &= ~(1ull << (8 * ay + ax));
      if (move) {
        // a3's front cell before the motion: not clear unless empty and no
        // ball (a free bit: the agent's own cell is not in front of it) or the
        // goal (never under a ball)
        const int fx = ax + (dir == 0 ? 1 : dir == 2 ? -1 : 0), fy = ay + (dir == 1 ? 1 : dir == 3 ? -1 : 0);
        const uint8_t f0 = g.get(fx, fy);
        not_clear_pre = (f0 & 15) != K_GOAL && !((freeb >> (8 * fy + fx)) & 1ull);
      }
      // generation: (env, episode, 0, block 0); transition: (env, episode, 1 << 16 | step, 0)
      const uint4 u = philox4x32_10(make_uint4(genv, episode, gen ? 0u : (1u << 16) | sc, 0u), a.key_lo, a.key_hi);
      // Generation needs no mask: the fixed start's free cells are the
      // interior minus the agent (1, 1) — the first interior cell — and the
      // goal (W-2, H-2) — the last —, i.e. interior cells 1 .. NFREE0 in
      // row-major order, and ball b is cell k_b of that list minus the cells
      // of the balls before it: one pass over their list indices in ascending
      // order (gs, kept sorted) steps k_b over each one at or below it.
      constexpr int IW = W - 2, NFREE0 = (W - 2) * (H - 2) - 2;
      static_assert(NFREE0 >= C::NOBST && C::NOBST <= 4, "never out of cells; the balls fit the low word");
      static_assert(template_free_cells<FAM, H, W>() == interior_cells<H, W>() - (1ull << (8 * (H - 2) + W - 2)),
                    "the template's free cells are the interior minus the goal");
      uint32_t gs[C::NOBST > 0 ? C::NOBST : 1];
      uint32_t b32 = (uint32_t)balls;  // byte b = ball b's bit index (0: none)
#pragma unroll
      for (int bb = 0; bb < C::NOBST; ++bb) {
        const uint32_t p = (b32 >> (8 * bb)) & 0xFF;
        const uint32_t ub = bb == 0 ? u.x : bb == 1 ? u.y : bb == 2 ? u.z : u.w;
        // transition: the 3x3 box around the ball, from bit 8 (by-1) + (bx-1)
        // = p - 9 (interior ball: p >= 9), as three 3-bit rows of a word
        const int sh = (int)p - 9;
        const uint32_t box = p ? (uint32_t)(freeb >> (sh & 63)) & 0x070707u : 0u;
        const uint32_t n = gen ? (uint32_t)(NFREE0 - bb) : (uint32_t)__popc(box);
        const uint32_t k = bounded(ub, n);  // k-th admissible cell, row-major
        int pos;
        if (gen) {
          uint32_t i = k;
#pragma unroll
          for (int j = 0; j < bb; ++j) i += gs[j] <= i ? 1u : 0u;
          if (bb + 1 < C::NOBST) {  // insert i into the sorted list
            uint32_t x = i;
#pragma unroll
            for (int j = 0; j < bb; ++j) {
              const uint32_t lo = min(gs[j], x);
              x = max(gs[j], x);
              gs[j] = lo;
            }
            gs[bb] = x;
          }
          const uint32_t q = i + 1u;  // interior cell q (0 = the agent's) = bit 9 + q + (8 - IW) (q / IW)
          pos = (int)(9u + q + (8u - IW) * (q / IW));
        } else {
          // the k-th set bit of the box: its row, then its column
          const uint32_t c0 = __popc(box & 0x7u), c1 = __popc(box & 0x707u);
          const bool ge0 = k >= c0, ge1 = k >= c1;
          const uint32_t r8 = (ge0 ? 8u : 0u) + (ge1 ? 8u : 0u);
          const uint32_t kr = k - (ge1 ? c1 : ge0 ? c0 : 0u);
          const uint32_t row = (box >> r8) & 0x7u;
          const uint32_t col = (kr >= (row & 1u) ? 1u : 0u) + (kr >= (uint32_t)__popc(row & 3u) ? 1u : 0u);
          pos = sh + (int)(r8 + col);
        }
        if (n) {  // (always for generation: NFREE0 >= NOBST)
          if (!gen) freeb = (freeb | (1ull << p)) & ~(1ull << pos);  // the old cell is empty now
          b32 = __byte_perm(b32, (uint32_t)pos, (0x3210u & ~(0xFu << (4 * bb))) | (4u << (4 * bb)));
        }
      }
      balls = b32;
      const uint32_t fails = 0;
      if (gen) st_fail = fails;
      if (scratch != nullptr && balls != balls_before) {
        // rollout: the SMEM rows persist across steps and hold last step's
        // balls; their cells are empty in the static layout
#pragma unroll
        for (int bb = 0; bb < C::NOBST; ++bb) {
          const uint32_t p = (uint32_t)(balls_before >> (8 * bb)) & 0xFF;
          if (p) g.set(ball_x(W, p), ball_y(W, p), CELL_EMPTY);
        }
      }
    }
    if (!regen || gen) overlay_balls();  // (queue-generated levels already hold theirs)
  }
  // Dynamic-Obstacles draws of this step, one Philox block per 4 balls:
  // generation (env, episode, 0, block) — the level generator's stream —,
  // transition (env, episode, 1 << 16 | step, block)
  constexpr int DYN_NB = UNIFIED_ROWS ? (C::NOBST + 3) / 4 : 1;
  uint4 dyn_u[DYN_NB];
  if constexpr (UNIFIED_ROWS) {
    const bool gen = unified && regen;
    if (gen) {
      // a2 (R#18): episode e+1 of [MG] DynamicObstaclesEnv, agent (1,1) east
      episode = (in.episode_known ? episode : a.episode[slot]) + 1u;
      ax = 1; ay = 1; dir = 0;
      carry = CELL_EMPTY;
      sc = 0;
      prev_done = false;
      if (!grid_tmpl) {  // an imported layout: back to the template (SMEM now, HBM at write-back)
#pragma unroll
        for (int q = 0; q < H * RW; ++q) rows[q * TILE] = template_plane<FAM, H, W>(q);
      } else if (in.rows_persist) {
        // rollout: the SMEM rows persist across steps and hold the last
        // episode's balls; their cells are empty in the static layout
#pragma unroll
        for (int bb = 0; bb < C::NOBST; ++bb) {
          const uint32_t p = (uint32_t)(balls >> (8 * bb)) & 0xFF;
          if (p) g.set(ball_x(W, p), ball_y(W, p), CELL_EMPTY);
        }
      }
      grid_dirty = !grid_tmpl;
      grid_tmpl = true;
      st_fail = 0;
    }
    if (gen || !regen) {
#pragma unroll
      for (int k = 0; k < DYN_NB; ++k)
        dyn_u[k] = philox4x32_10(make_uint4(genv, episode, gen ? 0u : (1u << 16) | sc, (uint32_t)k), a.key_lo, a.key_hi);
    }
    if (gen) {
      // the fixed start's free cells are interior cells 1 .. NFREE0 in
      // row-major order (0 is the agent's, the last the goal's); ball b is
      // cell k_b of that list minus those of the balls before it (one pass
      // over their list indices gs, kept sorted, as the BITBOARD loop)
      constexpr int IW = W - 2, NFREE0 = (W - 2) * (H - 2) - 2;
      static_assert(NFREE0 >= C::NOBST, "the generator never runs out of cells here");
      uint32_t gs[C::NOBST > 0 ? C::NOBST : 1];
      balls = 0;
#pragma unroll
      for (int bb = 0; bb < C::NOBST; ++bb) {
        const uint4& x = dyn_u[bb >> 2];
        const uint32_t ub = (bb & 3) == 0 ? x.x : (bb & 3) == 1 ? x.y : (bb & 3) == 2 ? x.z : x.w;
        uint32_t i = bounded(ub, (uint32_t)(NFREE0 - bb));
#pragma unroll
        for (int j = 0; j < bb; ++j) i += gs[j] <= i ? 1u : 0u;
        if (bb + 1 < C::NOBST) {
          uint32_t v = i;
#pragma unroll
          for (int j = 0; j < bb; ++j) {
            const uint32_t lo = min(gs[j], v);
            v = max(gs[j], v);
            gs[j] = lo;
          }
          gs[bb] = v;
        }
        const uint32_t q = i + 1u;  // interior cell q
        const int bx = 1 + (int)(q % IW), by = 1 + (int)(q / IW);
        balls |= (uint64_t)ball_code(W, bx, by) << (8 * bb);
      }
      overlay_balls();
    }
  }
  if (!regen) {
    if (FAM == FAM_DYNOBS && !BITBOARD) overlay_balls();
    if (MODE == MODE_STEP) {
      const int dx = dir == 0 ? 1 : dir == 2 ? -1 : 0;
      const int dy = dir == 1 ? 1 : dir == 3 ? -1 : 0;
      const int fx = ax + dx, fy = ay + dy;
      bool not_clear = false;
      if constexpr (BITBOARD) {
        not_clear = not_clear_pre;  // a3 ran above
      } else if (FAM == FAM_DYNOBS) {
        // ---- a3: transition mu (R#4, R#5, R#7)
        if (act >= 3) act = 0;
        const uint8_t f0 = g.get(fx, fy);
        not_clear = f0 != CELL_EMPTY && (f0 & 15) != K_GOAL;
        // one Philox block per 4 balls: (env, episode, 1 << 16 | step, block)
        uint4 u = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int bb = 0; bb < C::NOBST; ++bb) {
          if ((bb & 3) == 0) {
            if constexpr (UNIFIED_ROWS) u = dyn_u[bb >> 2];  // drawn above
            else u = philox4x32_10(make_uint4(genv, episode, (1u << 16) | sc, (uint32_t)(bb >> 2)), a.key_lo, a.key_hi);
          }
          const uint32_t p = (uint32_t)(balls >> (8 * bb)) & 0xFF;
          if (!p) continue;
          const int bx = p >> 4, by = p & 15;
          // admissible cells of the 3x3 box, row-major bit k = 4*dy + dx: empty
          // (cell byte == 0x01) and not the agent
          uint32_t m = 0;
          if constexpr (RW == 1) {
            // a byte permute gathers the 3 cells of each row, a SWAR exact-zero
            // test finds the empty ones
            const uint32_t sel = (uint32_t)((bx - 1) | (bx << 4) | ((bx + 1) << 8));
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const uint64_t line = rows[(by - 1 + dy) * TILE];
              const uint32_t x = prmt((uint32_t)line, (uint32_t)(line >> 32), sel) ^ 0x01010101u;
              const uint32_t z = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);  // bit 7: byte == 0
              m |= (((z & 0x00808080u) * 0x00204080u) >> 28) << (4 * dy);
            }
          } else {
            // wide rows: the 3 cells x = bx-1 .. bx+1 of a row from one or two
            // 32-bit words (a funnel shift), then the same SWAR empty test
            const int x0 = bx - 1, k = x0 >> 2, sh = 8 * (x0 & 3);
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int y = by - 1 + dy;
              const uint32_t* w = reinterpret_cast<const uint32_t*>(rows + (y * RW + (k >> 1)) * TILE) + (k & 1);
              const uint32_t w0 = *w;
              const uint32_t* w1p = reinterpret_cast<const uint32_t*>(rows + (y * RW + ((k + 1) >> 1)) * TILE) +
                                    ((k + 1) & 1);
              const uint32_t w1 = (x0 & 3) > 1 ? *w1p : 0u;  // only when the 3 cells straddle two words
              const uint32_t x = (__funnelshift_r(w0, w1, sh) & 0x00FFFFFFu) ^ 0x01010101u;
              const uint32_t z = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x | 0x7F7F7F7Fu);
              m |= (((z & 0x00808080u) * 0x00204080u) >> 28) << (4 * dy);
            }
          }
          const int adx = ax - (bx - 1), ady = ay - (by - 1);
          if ((unsigned)adx < 3u && (unsigned)ady < 3u) m &= ~(1u << (4 * ady + adx));
          if (m) {
            const uint32_t ub = (bb & 3) == 0 ? u.x : (bb & 3) == 1 ? u.y : (bb & 3) == 2 ? u.z : u.w;
            // the k-th set bit (row-major order): its row (two prefix
            // popcounts of the 4-bit rows), then its column
            const uint32_t k = bounded(ub, __popc(m));
            const uint32_t c0 = __popc(m & 0xFu), c1 = __popc(m & 0xFFu);
            const bool ge0 = k >= c0, ge1 = k >= c1;
            const uint32_t r = (ge0 ? 1u : 0u) + (ge1 ? 1u : 0u);
            const uint32_t kr = k - (ge1 ? c1 : ge0 ? c0 : 0u);
            const uint32_t row = (m >> (4 * r)) & 0x7u;
            const uint32_t col = (kr >= (row & 1u) ? 1u : 0u) + (kr >= (uint32_t)__popc(row & 3u) ? 1u : 0u);
            const int nx = bx - 1 + (int)col, ny = by - 1 + (int)r;
            g.set(nx, ny, make_cell(K_BALL, COL_BLUE));
            g.set(bx, by, CELL_EMPTY);
            // ball byte bb = ball_code (x << 4 | y on these grids): one byte
            // permute on the word holding it
            const uint32_t code = ((uint32_t)nx << 4) | (uint32_t)ny;
            const uint32_t SEL = (0x3210u & ~(0xFu << (4 * (bb & 3)))) | (4u << (4 * (bb & 3)));
            if (bb < 4) balls = (balls & 0xFFFFFFFF00000000ull) | __byte_perm((uint32_t)balls, code, SEL);
            else balls = (balls & 0xFFFFFFFFull) | ((uint64_t)__byte_perm((uint32_t)(balls >> 32), code, SEL) << 32);
          }
        }
      }
      // ---- a4: intervention I (Table 3; [MG] MiniGridEnv.step), branch-free:
      // every action's effect is computed with selects so a warp never splits
      // on the action value.
      sc += 1;
      uint8_t* fp = g.at(fx, fy);
      // GoToDoor's grid edge is open: outside the grid reads as a wall (R#37)
      const bool f_out = FAM == FAM_GOTODOOR && ((unsigned)fx >= (unsigned)W || (unsigned)fy >= (unsigned)H);
      const uint32_t fc = f_out ? (uint32_t)CELL_WALL : *fp;
      const uint32_t kind = fc & 15u;
      // (Dynamic-Obstacles maps every action >= 3 to left, R#7: no pickup,
      // drop or toggle can happen, and the compiler drops their logic)
      constexpr bool MANIP = FAM != FAM_DYNOBS;
      const bool is_fwd = act == 2, is_pick = MANIP && act == 3, is_drop = MANIP && act == 4,
                 is_tog = MANIP && act == 5;
      dir = (dir + (act == 1 ? 1 : 0) + (act == 0 ? 3 : 0)) & 3;
      const bool walk = (0x31Au >> kind) & 1u;  // empty, floor, open door, goal, lava
      ax = (is_fwd && walk) ? fx : ax;
      ay = (is_fwd && walk) ? fy : ay;
      bool success = is_fwd && kind == K_GOAL;
      bool lava = is_fwd && kind == K_LAVA;
      bool coll = false;
      const bool pick = is_pick && ((0xE0u >> kind) & 1u) && carry == CELL_EMPTY;  // key, ball, box
      const bool drop = is_drop && fc == CELL_EMPTY && carry != CELL_EMPTY;
      // [MG] Door.toggle / Box.toggle
      const uint32_t colbits = fc & 0x70u;
      const bool key_ok = (carry & 15u) == K_KEY && (carry & 0x70u) == colbits;
      const uint32_t opened = colbits | K_DOOR_OPEN, closed = OPAQUE_BIT | colbits | K_DOOR_CLOSED;
      const uint32_t tog = ((kind == K_DOOR_LOCKED && key_ok) || kind == K_DOOR_CLOSED) ? opened
                           : kind == K_DOOR_OPEN ? closed
                           : kind == K_BOX ? (uint32_t)CELL_EMPTY : fc;
      const uint32_t newf = pick ? (uint32_t)CELL_EMPTY : drop ? (uint32_t)carry : is_tog ? tog : fc;
      carry = pick ? (uint8_t)fc : drop ? CELL_EMPTY : carry;
      if (newf != fc) {
        *fp = (uint8_t)newf;
        dirty_plane = fy * RW + (fx >> 3);
        grid_dirty = true;
        grid_tmpl = false;  // no longer the template layout
        room_closed = false;  // GoToDoor: a door opened
      }
      if (FAM == FAM_KEYCORRIDOR && is_pick && (carry & 15) == K_BALL) success = true;  // R#8
      if (FAM == FAM_DYNOBS && is_fwd && not_clear) { coll = true; success = false; }  // R#4
      bool gtd_end = false;
      if (FAM == FAM_GOTODOOR) {
        // [MG] GoToDoorEnv.step: toggle ends the episode; done ends it, a
        // success iff the agent is next to the target door (R#37).  Navix
        // reward mode: Table 6/7 `on_door_done`, done in front of the target
        // door is the only event (R#39)
        const int tx = (int)(target >> 4), ty = (int)(target & 15);
        const int ddx = ax - tx, ddy = ay - ty;
        const bool nav = a.reward_mode == 1;
        const bool hit = nav ? (fx == tx && fy == ty) : ddx * ddx + ddy * ddy == 1;
        gtd_end = !nav && (is_tog || act == 6);
        success = success || (act == 6 && hit);
        coll = gtd_end && !success;  // counted as n_failure, reward 0
      }
      // ---- a5: reward and termination (Eq. 1, Tables 6-7).
      // The events are exclusive; the Table 6 / 7 selection (R#42) decides
      // which of them pay their reward and which end the episode.
      const uint32_t ev = success ? 1u : coll ? 4u : lava ? 2u : 0u;  // a collision into lava counts as collision
      const uint32_t pay = ev & a.reward_events;
      if (pay == 4u && FAM != FAM_GOTODOOR) reward = -1.0f;
      else if (__builtin_expect(pay == 1u, 0)) reward = success_reward(a.reward_mode, sc, C::T);
      else if (pay == 2u) reward = a.reward_mode == 1 ? -1.0f : 0.0f;
      if (!(ev & a.termination_events)) success = lava = coll = false;
      // Code 4 `compose`: + (-time_cost) every step, + (-action_cost) for every
      // action but done, in binary32 in this order (R#31)
      if (a.time_cost != 0.f || a.action_cost != 0.f) {
        reward = __fadd_rn(reward, -a.time_cost);
        reward = __fadd_rn(reward, act != 6 ? -a.action_cost : 0.f);
      }
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

  // ---- a7a: grid write-back (only when modified), before the lines are reused
  // (pickup / drop / toggle change one cell: only its 8-byte plane is written,
  // one 32-byte sector instead of H*RW of them)
  if (MODE != MODE_OBSERVE && grid_dirty && scratch == nullptr) {
    uint64_t* gdst = a.grid + tile0 * H * RW + tid;
    const int wl = (int)(threadIdx.x % WIDE_LANES);  // WIDE: lane wl writes planes p = wl mod WIDE_LANES
    if (FAM != FAM_DYNOBS && dirty_plane >= 0) {
      if (!WIDE || wl == 0) gdst[dirty_plane * TILE] = rows[dirty_plane * TILE];
    } else {
#pragma unroll
      for (int p = 0; p < H * RW; ++p)
        if (!WIDE || p % WIDE_LANES == wl)
          gdst[p * TILE] = FAM == FAM_DYNOBS ? template_plane<FAM, H, W>(p) : rows[p * TILE];
    }
  }
  if constexpr (WIDE) {  // the observation is split over the lanes by the caller
    EnvResult r;
    r.reward = reward;
    r.valid = valid;
    r.regen = regen;
    r.term = term;
    r.trunc = trunc;
    r.dirty = grid_dirty;
    r.tvalid = false;
    r.nrec = (uint64_t)(uint32_t)ax | ((uint64_t)(uint32_t)ay << 8) | ((uint64_t)dir << 16) |
             ((uint64_t)carry << 24) | ((uint64_t)sc << 32) | ((uint64_t)(prev_done ? 1 : 0) << 48) |
             ((uint64_t)(grid_tmpl ? 1 : 0) << 49) | ((uint64_t)(layout_key || room_closed ? 1 : 0) << 50) | ((uint64_t)target << 56);
    r.episode = episode;
    r.balls = balls;
    const uint32_t vv = valid && (threadIdx.x % WIDE_LANES) == 0 ? 1u : 0u;  // counted once per env
    r.st[0] = st_ep * vv; r.st[1] = st_len * vv; r.st[2] = st_succ * vv; r.st[3] = st_succ_len * vv;
    r.st[4] = st_lava * vv; r.st[5] = st_coll * vv; r.st[6] = st_trunc * vv; r.st[7] = st_fail * vv;
    return r;
  }

  // ---- a6: observation (obs.cuh); odd directions read world columns
  // Dynamic-Obstacles on its static layout (the whole warp): balls are
  // see-through ([MG] Ball), so the visibility mask depends on the agent pose
  // alone and comes from a per-pose table (obs_table_kernel) instead of the
  // opacity gather and the row closures
  // (DoorKey: a table per layout key, LAYOUT_KEYED_VIS)
  constexpr bool VIS_TABLE = (STATIC_LAYOUT<FAM> || KEYED_VIS) && !WIDE;
  bool table_vis = false;
  uint32_t tvis_lo = 0, tvis_hi = 0;
  if constexpr (VIS_TABLE) {
    table_vis = __all_sync(0xffffffffu, !valid || (KEYED_VIS ? layout_key : grid_tmpl));
    if (table_vis && valid) {
      int layout = 0;
      if constexpr (LAYOUT_KEYED_VIS<FAM, W>) {  // read before odd directions transpose the rows
        const int split = (int)(target >> 4), door_y = (int)(target & 15);
        const bool open = (g.get(split, door_y) & 15) == K_DOOR_OPEN;
        layout = (((split - 2) * (W - 3) + (door_y - 1)) << 1) | (open ? 1 : 0);
      }
      // issued early: its latency hides behind the transpose and the view
      // columns (a load next to its use measured 2 % slower, 42.2 vs 41.3 us)
      const uint2 v = __ldg(obs_table_entry<FAM, H, W>(ax, ay, dir, layout));
      tvis_lo = v.x;
      tvis_hi = v.y;
    }
  }
  const uint64_t* lines = rows;
  // rollout: the transposed lines stay valid while the grid does not change
  // (Dynamic-Obstacles moves its balls every step: never cached)
  bool tvalid = FAM != FAM_DYNOBS && scratch != nullptr && in.tvalid && !grid_dirty;
  if (RW == 1 && (dir & 1)) {
    if (scratch) {
      if (!tvalid) transpose_lines(rows, scratch);
      tvalid = FAM != FAM_DYNOBS;
      lines = scratch;
    } else {
      transpose_lines(rows, rows);
    }
  }
  before_emit();
  {
    uint32_t* const s32 = reinterpret_cast<uint32_t*>(s_obs);
    constexpr int OB = obs_record_bytes(OBSK);
    // warp-uniform record misalignment: 147*le mod 4 = 3w mod 4, 49*le mod 4 = w
    const int M = OBSK == OBS_CATEGORICAL ? warp & 3 : (3 * warp) & 3;
    uint32_t clo[7], chi[7];
    if constexpr (RW == 1) view_columns_narrow(lines, ax, ay, dir, clo, chi);
    else view_columns_big<RW, H>(rows, ax, ay, dir, clo, chi);
    if constexpr (FAM == FAM_GOTODOOR) {
      if (!room_closed) view_oob_walls<H, W>(ax, ay, dir, clo, chi);  // R#37
    }
    uint32_t vis_lo, vis_hi;
    if (table_vis) {
      vis_lo = tvis_lo;
      vis_hi = tvis_hi;
    } else {
      view_visibility(clo, chi, vis_lo, vis_hi);
    }
    if constexpr (OBSK == OBS_CATEGORICAL) observe_cols_cat(clo, chi, carry, s32 + ((le * OB - M) >> 2), M, vis_lo, vis_hi);
    else observe_cols(clo, chi, carry, s32 + ((le * OB - M) >> 2), M, vis_lo, vis_hi);
  }

  EnvResult r;
  r.reward = reward;
  r.valid = valid;
  r.regen = regen;
  r.term = term;
  r.trunc = trunc;
  r.dirty = grid_dirty;
  r.tvalid = tvalid;
  r.nrec = (uint64_t)(uint32_t)ax | ((uint64_t)(uint32_t)ay << 8) | ((uint64_t)dir << 16) | ((uint64_t)carry << 24) |
           ((uint64_t)sc << 32) | ((uint64_t)(prev_done ? 1 : 0) << 48) | ((uint64_t)(grid_tmpl ? 1 : 0) << 49) | ((uint64_t)(layout_key || room_closed ? 1 : 0) << 50) |
           ((uint64_t)target << 56);
  r.episode = episode;
  r.balls = balls;
  const uint32_t vv = valid ? 1u : 0u;
  r.st[0] = st_ep * vv; r.st[1] = st_len * vv; r.st[2] = st_succ * vv; r.st[3] = st_succ_len * vv;
  r.st[4] = st_lava * vv; r.st[5] = st_coll * vv; r.st[6] = st_trunc * vv; r.st[7] = st_fail * vv;
  return r;
}

// a7: the tile's obs leave SMEM in one TMA bulk store (full tile, 16-B aligned
// destination) issued by one thread, else with plain stores by `nthr` threads.
template <int OBSK>
__device__ __forceinline__ void store_obs(const KernelArgs& a, int64_t tile, const uint8_t* s_obs, int t, int nthr,
                                          bool issuer) {
  constexpr int OB = obs_record_bytes(OBSK);
  const int64_t tile0 = tile * TILE;
  const int64_t nv = a.n - tile0;
  const int nvalid = nv >= TILE ? TILE : (int)nv;
  uint8_t* dst = a.obs + tile0 * OB;
  if (a.bulk_obs && nvalid == TILE) {
    if (issuer) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(s_obs)),
                   "r"((uint32_t)(TILE * OB))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  } else {
    for (int i = t; i < nvalid * OB; i += nthr) dst[i] = s_obs[i];
  }
}

// a7: per-env global stores and the episode statistics (WRITE_STATE = 0 in a
// rollout, whose state stays on chip until its last step).
// Episode statistics of the envs a thread stepped, summed in registers over
// the tiles of a persistent / rollout CTA and flushed once (warp reduce ->
// striped int64 atomics) instead of once per tile.
struct StatsAcc {
  uint32_t v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  __device__ __forceinline__ void add(const EnvResult& r) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] += r.st[k];
  }
  __device__ __forceinline__ void flush(const KernelArgs& a) const {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t any = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) any |= v[k];
    if (!__any_sync(0xffffffffu, any != 0)) return;
    uint32_t w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = __reduce_add_sync(0xffffffffu, v[k]);
    if (lane == 0) {
      unsigned long long* st = a.stats + (size_t)((blockIdx.x * (TILE / 32) + warp) % NSLOT) * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (w[k]) atomicAdd(st + k, (unsigned long long)w[k]);
    }
  }
};

template <int FAM, int MODE, bool WRITE_STATE = true, bool STATS = true>
__device__ __forceinline__ void tile_store(const KernelArgs& a, int64_t tile, const EnvResult& r) {
  if (MODE == MODE_OBSERVE) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t slot = tile * TILE + tid, e = tile * TILE + 4 * lane + warp;
  if (r.valid) {
    if (MODE == MODE_STEP) {
      a.reward[e] = r.reward;
      a.terminated[e] = r.term;
      a.truncated[e] = r.trunc;
    }
    if (WRITE_STATE) {
      a.agent[slot] = r.nrec;
      if (r.regen) a.episode[slot] = r.episode;
      if (FAM == FAM_DYNOBS) a.balls[slot] = r.balls;
    }
  }
  // episode statistics (info i_{t+1}): warp reduce -> striped atomics
  if (!STATS) return;  // accumulated by the caller (StatsAcc)
  const unsigned any = __any_sync(0xffffffffu, (r.st[0] | r.st[7]) != 0);
  if (any) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __reduce_add_sync(0xffffffffu, r.st[k]);
    if (lane == 0) {
      unsigned long long* st = a.stats + (size_t)((tile * (TILE / 32) + warp) % NSLOT) * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (v[k]) atomicAdd(st + k, (unsigned long long)v[k]);
    }
  }
}

// ------------------------------------------------------------------ kernels
// One tile per CTA (reset, observe; step when NAVIX_STEP_KERNEL=onetile).
// 28 KB of SMEM: up to 8 CTAs per SM with <= 64 registers.
template <int FAM, int NPL, int OBSK>
struct OneTileSmem {
  uint8_t obs[TILE * obs_record_bytes(OBSK)];
  TileSmem<FAM, NPL> buf;
  uint64_t scratch[NPL == 8 ? 8 : 1][TILE];  // rollout: column view of odd directions (narrow grids)
  uint64_t mbar;
};
extern __shared__ __align__(128) uint8_t navix_dyn_smem[];

template <int FAM, int H, int W, int MODE, int OBSK>
__global__ void __launch_bounds__(TILE, (W > 8 ? 3 : 8)) navix_kernel(const KernelArgs a) {
  using C = Cfg<FAM, H, W>;
  auto& S = *reinterpret_cast<OneTileSmem<FAM, C::NPL, OBSK>*>(navix_dyn_smem);
  if (MODE == MODE_STEP) {  // launched with programmatic dependent launch (see navix_step_persistent)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  if (MODE != MODE_RESET) {
    const uint32_t mbar = smem_u32(&S.mbar);
    if (MODE == MODE_STEP) init_reset_queue_counter<FAM>();
    if (threadIdx.x == 0) {
      mbar_init(mbar, 1);
      issue_tile_loads<FAM, H * C::RW, MODE>(a, blockIdx.x, S.buf, mbar);
    }
    __syncthreads();  // mbarrier initialised before anyone waits on it
    mbar_wait(mbar, 0);
  }
  const EnvResult r = tile_compute<FAM, H, W, MODE, OBSK>(a, blockIdx.x, &S.buf.rows[0][threadIdx.x], nullptr,
                                                    decode_staged<FAM, MODE>(a, blockIdx.x, S.buf), S.obs, [] {});
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  store_obs<OBSK>(a, blockIdx.x, S.obs, threadIdx.x, TILE, threadIdx.x == 0);
  tile_store<FAM, MODE>(a, blockIdx.x, r);
  // exit once the bulk store has READ the staging buffer; its global writes
  // complete with the grid (the TMA-store epilogue idiom)
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// Persistent step: each CTA pulls tiles from a global atomic scheduler and
// keeps the next tile's inputs in flight (TMA, double-buffered, mbarrier-
// tracked) while it computes the current one.  Per tile: one CTA barrier after
// the obs emission (thread 0 then issues the tile's TMA store and the
// prefetch of the tile-after-next into the released input buffer) and one
// before the next tile's emission, by which time the store has long read the
// staging buffer.  The scheduler atomic is issued a whole tile early.  (A barrier-free
// variant where the last warp to finish issues the store measured 1.3 % slower:
// its warps spin on mbarriers instead.)  The last CTA to finish resets the
// scheduler, so the kernel replays from a CUDA graph.
template <int FAM, int NPL, int OBSK>
struct PersistSmem {
  uint8_t obs[TILE * obs_record_bytes(OBSK)];
  TileSmem<FAM, NPL> buf[2];
  uint64_t mbar[2];  // tile inputs landed (per buffer)
  int64_t tile[2];
};

template <int FAM, int H, int W, int OBSK>
__global__ void __launch_bounds__(TILE) navix_step_persistent(const KernelArgs a) {
  using C = Cfg<FAM, H, W>;
  auto& S = *reinterpret_cast<PersistSmem<FAM, C::NPL, OBSK>*>(navix_dyn_smem);
  uint8_t* const s_obs = S.obs;
  auto& s_buf = S.buf;
  auto& s_mbar = S.mbar;
  auto& s_tile = S.tile;
  const int64_t n_tiles = (a.n + TILE - 1) / TILE;
  unsigned int* const sched = a.sched;          // [0] ticket, [1] CTAs done, [2] epoch, [3..4] list counts
  unsigned int* const marks = sched + 8;        // [2][n_tiles] epoch stamps, then [2][n_tiles] lists
  const int tid = threadIdx.x;
  // fetch the next tile index into s_tile[k] and start its loads on s_mbar[k];
  // with no tile left only arrive (the phase completes), so waiting on
  // s_mbar[k] always publishes s_tile[k].
  auto publish = [&](int k, int64_t t) {
    s_tile[k] = t;
    if (t < n_tiles) issue_tile_loads<FAM, H * C::RW, MODE_STEP>(a, t, s_buf[k], smem_u32(&s_mbar[k]));
    else mbar_arrive(smem_u32(&s_mbar[k]));
  };
  // Programmatic dependent launch: let the next step's grid be scheduled now
  // (its CTAs take the SM slots ours free and wait below), and wait for the
  // previous step's grid to complete and flush before touching global memory.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // small batches (<= 4 tiles per CTA): plain striding, no scheduler atomics
  // on the critical path; larger ones balance with the atomic counter
  constexpr bool RESET_FIRST_FAM = FAM == FAM_KEYCORRIDOR;
  // KeyCorridor keeps the dynamic scheduler whenever a CTA gets more than one
  // tile: in steady state (desynchronised episodes, ~1/270 of the envs reset
  // every step) a third of the tiles carry a long level generation, and
  // claiming those first balances them over the CTAs (striding stacked up to
  // four of them on one CTA)
  const bool stride_only = n_tiles <= (RESET_FIRST_FAM ? 1 : 4) * (int64_t)gridDim.x;
  if (tid == 0) {
    mbar_init(smem_u32(&s_mbar[0]), 1);
    mbar_init(smem_u32(&s_mbar[1]), 1);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // Tiles with envs that auto-reset this step (marked by the previous step)
  // go first: their level generation (a long serial chain for KeyCorridor)
  // then overlaps the other tiles instead of trailing the step.  Ticket t <
  // L takes the t-th listed tile, later tickets the tiles in index order,
  // skipping listed ones.  Epoch stamps make the marks self-clearing.
  // (stamps and lists are double-buffered by epoch parity: this step reads
  // the previous step's, and writes the next step's, so a stamp never
  // changes while it is read)
  // Only KeyCorridor uses it: its resets are rare but each is a long serial
  // level generation; families that reset often gain nothing and would pay
  // the stamp reads and list atomics.
  // (striding, the small-batch mode, has no claim order to change: off there;
  // the mode is fixed for a handle, so the lists stay consistent)
  const bool RESET_FIRST = RESET_FIRST_FAM && !stride_only;
  const uint32_t epoch = RESET_FIRST ? sched[2] : 0u;
  const uint32_t L = RESET_FIRST ? sched[3 + (epoch & 1u)] : 0u;
  const unsigned int* mark_cur = marks + (epoch & 1u) * n_tiles;
  unsigned int* const mark_next = marks + ((epoch + 1u) & 1u) * n_tiles;
  const unsigned int* list_cur = marks + 2 * n_tiles + (epoch & 1u) * n_tiles;
  unsigned int* const list_next = marks + 2 * n_tiles + ((epoch + 1u) & 1u) * n_tiles;
  auto ticket_tile = [&](uint32_t t) -> int64_t {  // thread 0
    if (!RESET_FIRST) return (int64_t)t;
    for (;;) {
      if (t < L) return (int64_t)list_cur[t];
      const int64_t tile = (int64_t)(t - L);
      if (tile >= n_tiles || mark_cur[tile] != epoch + 1u) return tile;
      t = atomicAdd(&sched[0], 1u) + 2u * gridDim.x;  // listed: already someone's
    }
  };
  init_reset_queue_counter<FAM>();
  if (tid == 0) {
    // the first two tickets are static (b, b + grid): no burst of contended
    // atomics on the scheduler word when every CTA starts at once
    publish(0, ticket_tile(blockIdx.x));
    publish(1, ticket_tile(blockIdx.x + gridDim.x));
  }
  __syncthreads();
  StatsAcc acc;
  for (int it = 0;; ++it) {
    const int cur = it & 1;
    mbar_wait(smem_u32(&s_mbar[cur]), (uint32_t)(it >> 1) & 1u);
    const int64_t tile = s_tile[cur];
    if (tile >= n_tiles) break;
    // claim the tile-after-next now: the atomic's latency hides behind the compute
    unsigned int next = 0;
    if (tid == 0) next = stride_only ? (unsigned)(tile + 2 * gridDim.x) : atomicAdd(&sched[0], 1u) + 2u * gridDim.x;
    const EnvResult r = tile_compute<FAM, H, W, MODE_STEP, OBSK>(
        a, tile, &s_buf[cur].rows[0][tid], nullptr, decode_staged<FAM, MODE_STEP>(a, tile, s_buf[cur]), s_obs, [&] {
      if (it > 0) {  // the previous tile's store must have read s_obs
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
      }
    });
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // all records in s_obs; input buffer cur no longer read
    store_obs<OBSK>(a, tile, s_obs, tid, TILE, tid == 0);
    if (tid == 0) publish(cur, ticket_tile(next));  // tile-after-next into the released buffer
    tile_store<FAM, MODE_STEP, true, false>(a, tile, r);
    acc.add(r);
    // envs that ended reset at the next step: list their tile for it (once)
    if (RESET_FIRST && __any_sync(0xffffffffu, r.valid && (r.term || r.trunc)) && (tid & 31) == 0 &&
        atomicExch(&mark_next[tile], epoch + 2u) != epoch + 2u)
      list_next[atomicAdd(&sched[3 + ((epoch + 1u) & 1u)], 1u)] = (unsigned int)tile;
  }
  acc.flush(a);
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // SMEM read; writes complete with the grid
  // Pure striding claims no tickets, so (outside KeyCorridor's epochs) there
  // is nothing to reset and no exit atomic on the small-batch critical path.
  if (tid == 0 && (RESET_FIRST || !stride_only)) {
    __threadfence();
    if (atomicAdd(&sched[1], 1u) == gridDim.x - 1) {  // last CTA: reset the scheduler
      atomicExch(&sched[0], 0u);
      atomicExch(&sched[1], 0u);
      if (RESET_FIRST) {
        atomicExch(&sched[3 + (epoch & 1u)], 0u);  // this step's list is consumed
        atomicExch(&sched[2], epoch + 1u);
      }
    }
  }
}

// Small batches (SURVEY §8d's 2^10-2^14 points, the paper's 2048 agents
// P:43): one step of n envs is a handful of tiles, so its time is one env's
// dependent chain, not bandwidth.  Here WIDE_LANES lanes
// share an env: they run its step logic redundantly (tile_compute<WIDE>),
// split the grid write-back, and each builds ONE view column of the
// observation (the visibility rows are OR-reduced over the lanes with
// shuffles), so the observation's ~500 dependent instructions become ~100.
// 16 envs per 128-thread CTA; records staged in SMEM and copied out by their
// warp with word stores.  Grids up to 8 wide with a closed border (not
// GoToDoor).  Bit-identical to navix_step_persistent (tests/test_gpu_wide.py).
constexpr int WIDE_EPC = TILE / WIDE_LANES;  // envs per CTA
// a6 + a7 of the small-batch kernels: lane j < 7 of an env builds view
// column vi = j of its observation (after the step in r), the visibility rows
// are OR-reduced over the env's lanes, each lane writes its column's record
// bytes to SMEM, and each warp copies its 4 envs' records (contiguous,
// 4-byte aligned) to a.obs.  Called by all lanes of the CTA, converged.
template <int FAM, int H, int W, int OBSK>
__device__ __forceinline__ void wide_observe_and_store(const KernelArgs& a, const EnvResult& r, const uint64_t* rows,
                                                       uint8_t* s_obs) {
  constexpr int OB = obs_record_bytes(OBSK);
  const int t = threadIdx.x, g = t / WIDE_LANES, j = t % WIDE_LANES;
  __syncwarp();  // the warp's previous copy-out (rollout) has read s_obs
  // ---- a6 split by view column: lane j < 7 builds column vi = j
  const int ax = (int)(r.nrec & 0xFF), ay = (int)((r.nrec >> 8) & 0xFF), dir = (int)((r.nrec >> 16) & 3);
  const uint32_t carry = (uint32_t)((r.nrec >> 24) & 0xFF);
  uint32_t clo = 0, chi = 0;
  if (j < 7) view_column_narrow(rows, ax, ay, dir, j, clo, chi);
  const int js = j < 7 ? j : 0;
  uint32_t vis_lo, vis_hi;
  // the per-pose visibility tables (static layouts, DoorKey, border-only
  // opacity) when the whole warp qualifies; else the lanes' opacity columns
  // are OR-reduced and closed
  constexpr bool KEYED = LAYOUT_KEYED_VIS<FAM, W> || BORDER_OPACITY<FAM>;
  constexpr bool TABLE = STATIC_LAYOUT<FAM> || KEYED;
  const bool valid = (int64_t)blockIdx.x * WIDE_EPC + g < a.n;
  const bool flagged = ((r.nrec >> (KEYED ? 50 : 49)) & 1) != 0;
  if (TABLE && __all_sync(0xffffffffu, !valid || flagged)) {
    int layout = 0;
    if constexpr (LAYOUT_KEYED_VIS<FAM, W>) {
      const int split = (int)(r.nrec >> 60), door_y = (int)((r.nrec >> 56) & 15);
      const bool open = (reinterpret_cast<const uint8_t*>(rows)[door_y * TILE * 8 + split] & 15) == K_DOOR_OPEN;
      layout = valid ? (((split - 2) * (W - 3) + (door_y - 1)) << 1) | (open ? 1 : 0) : 0;
    }
    const uint2 v = valid ? __ldg(obs_table_entry<FAM, H, W>(ax, ay, dir, layout)) : make_uint2(0u, 0u);
    vis_lo = v.x;
    vis_hi = v.y;
  } else {
    uint32_t op_lo = j < 7 ? (clo >> (7 - js)) & (0x01010101u << js) : 0u;  // byte vj, bit vi: opaque
    uint32_t op_hi = j < 7 ? (chi >> (7 - js)) & (0x01010101u << js) : 0u;
#pragma unroll
    for (int k = 1; k < WIDE_LANES; k <<= 1) {  // OR over the env's lanes (aligned groups of 8)
      op_lo |= __shfl_xor_sync(0xffffffffu, op_lo, k);
      op_hi |= __shfl_xor_sync(0xffffffffu, op_hi, k);
    }
    visibility_closure(op_lo, op_hi, vis_lo, vis_hi);
  }
  if (j == 3) chi = prmt(chi, carry, 0x3410u);  // the agent sees what it carries (R#13)
  if (j < 7) {
    const uint32_t m_lo = prmt(vis_lo * (1u << (7 - js)), 0u, 0xBA98u);
    const uint32_t m_hi = prmt(vis_hi * (1u << (7 - js)), 0u, 0xBA98u);
    if constexpr (OBSK == OBS_CATEGORICAL) {
      const uint32_t tl = encode4_type(clo, m_lo), th = encode4_type(chi, m_hi);
      uint8_t* d = s_obs + g * OB + 7 * j;
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = (uint8_t)(tl >> (8 * k));
#pragma unroll
      for (int k = 0; k < 3; ++k) d[4 + k] = (uint8_t)(th >> (8 * k));
    } else {
      uint32_t rr[7];
      encode_col(clo, chi, m_lo, m_hi, 0u, rr);
      store_column_bytes(s_obs + g * OB + 21 * j, rr);
    }
  }
  __syncwarp();
  // ---- a7: each warp copies its 4 envs' records (contiguous, 4-byte aligned)
  {
    const int w = t >> 5, l = t & 31;
    const int64_t e0 = (int64_t)blockIdx.x * WIDE_EPC + 4 * w;
    const int64_t nv = a.n - e0;
    const int nbytes = (int)(nv <= 0 ? 0 : nv >= 4 ? 4 * OB : nv * OB);
    const uint8_t* src = s_obs + 4 * w * OB;
    uint8_t* dst = a.obs + e0 * OB;
    if ((reinterpret_cast<uintptr_t>(dst) & 3u) == 0) {
      const int nw = nbytes >> 2;
      for (int i = l; i < nw; i += 32)
        reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[i];
      for (int i = 4 * nw + l; i < nbytes; i += 32) dst[i] = src[i];
    } else {
      for (int i = l; i < nbytes; i += 32) dst[i] = src[i];
    }
  }
}


struct NoEmit {
  __device__ void operator()() const {}
};
template <int FAM, int H, int W, int OBSK>
__global__ void __launch_bounds__(TILE) navix_step_wide(const KernelArgs a) {
  using C = Cfg<FAM, H, W>;
  static_assert(C::RW == 1, "the small-batch kernel covers grids up to 8 wide");
  constexpr int OB = obs_record_bytes(OBSK);
  __shared__ __align__(16) uint64_t s_rows[8][TILE];  // env g's lines in column g (stride TILE, as RowViewT)
  __shared__ __align__(16) uint8_t s_obs[WIDE_EPC * OB];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int t = threadIdx.x, g = t / WIDE_LANES, j = t % WIDE_LANES;
  const int64_t e = (int64_t)blockIdx.x * WIDE_EPC + g;
  const bool valid = e < a.n;
  const int64_t tile = e / TILE;
  const int le = (int)(e % TILE), st = slot_of_env(le);
  const int64_t slot = tile * TILE + st;
  uint64_t* const rows = &s_rows[0][g];
  // inputs: lane j loads grid row j; every lane the agent record (one
  // broadcast transaction per env); padding envs get a legal dummy state
  EnvIn in{PADDING_AGENT_RECORD, 0u, 0ull, 0u, FAM == FAM_DYNOBS, false};
  if (j < H) rows[j * TILE] = valid ? a.grid[(tile * H + j) * TILE + st] : 0ull;
  if (valid) {
    in.rec = a.agent[slot];
    in.act = a.actions[e];
    if (FAM == FAM_DYNOBS) {
      in.balls = a.balls[slot];
      in.episode = a.episode[slot];
    }
  }
  __syncwarp();
  const EnvResult r = tile_compute<FAM, H, W, MODE_STEP, OBSK, NoEmit, true>(a, tile, rows, nullptr, in, nullptr,
                                                                          NoEmit{}, le);
  __syncwarp();
  wide_observe_and_store<FAM, H, W, OBSK>(a, r, rows, s_obs);
  if (valid && j == 0) {
    a.reward[e] = r.reward;
    a.terminated[e] = r.term;
    a.truncated[e] = r.trunc;
    a.agent[slot] = r.nrec;
    if (r.regen) a.episode[slot] = r.episode;
    if (FAM == FAM_DYNOBS) a.balls[slot] = r.balls;
  }
  StatsAcc acc;
  acc.add(r);
  acc.flush(a);
}

// f1 at small batches: K steps of 16 envs per CTA with 8 lanes per env (as
// navix_step_wide), the rows in SMEM and the agent record / episode / balls
// in registers across the K steps; bit-identical to K navix_step calls.
template <int FAM, int H, int W, int OBSK>
__global__ void __launch_bounds__(TILE) navix_rollout_wide(const KernelArgs a, int64_t K) {
  using C = Cfg<FAM, H, W>;
  static_assert(C::RW == 1, "the small-batch kernel covers grids up to 8 wide");
  constexpr int OB = obs_record_bytes(OBSK);
  __shared__ __align__(16) uint64_t s_rows[8][TILE];
  __shared__ __align__(16) uint8_t s_obs[WIDE_EPC * OB];
  const int t = threadIdx.x, g = t / WIDE_LANES, j = t % WIDE_LANES;
  const int64_t e = (int64_t)blockIdx.x * WIDE_EPC + g;
  const bool valid = e < a.n;
  const int64_t tile = e / TILE;
  const int le = (int)(e % TILE), st = slot_of_env(le);
  const int64_t slot = tile * TILE + st;
  uint64_t* const rows = &s_rows[0][g];
  EnvIn in{PADDING_AGENT_RECORD, 0u, 0ull, 0u, true, false};
  if (j < H) rows[j * TILE] = valid ? a.grid[(tile * H + j) * TILE + st] : 0ull;
  if (valid) {
    in.rec = a.agent[slot];
    in.episode = a.episode[slot];
    if (FAM == FAM_DYNOBS) in.balls = a.balls[slot];
  }
  const bool draw = a.actions == nullptr;  // in-kernel random policy (navix_rollout_random)
  const uint32_t genv = a.env_begin + (uint32_t)e;
  auto policy = [&](int64_t tt) -> uint32_t {
    const uint4 w = philox4x32_10(make_uint4(genv, a.act_t0 + (uint32_t)tt, 2u << 16, 0u), a.act_key_lo, a.act_key_hi);
    return bounded(w.x, (uint32_t)C::NA);
  };
  uint32_t next_act = !valid ? 0u : draw ? policy(0) : a.actions[e];
  bool dirty = false;
  StatsAcc acc;
  __syncwarp();
  for (int64_t k = 0; k < K; ++k) {
    in.act = next_act;
    if (k + 1 < K && valid) next_act = draw ? policy(k + 1) : a.actions[(k + 1) * a.n + e];  // one step ahead
    KernelArgs as = a;
    as.obs = a.obs + k * a.n * OB;
    as.reward = a.reward + k * a.n;
    as.terminated = a.terminated + k * a.n;
    as.truncated = a.truncated + k * a.n;
    // a non-null scratch: the rows stay in SMEM (no per-step grid write-back;
    // Dynamic-Obstacles clears its balls' old cells there)
    const EnvResult r = tile_compute<FAM, H, W, MODE_STEP, OBSK, NoEmit, true>(
        as, tile, rows, reinterpret_cast<uint64_t*>(s_obs), in, nullptr, NoEmit{}, le);
    __syncwarp();
    wide_observe_and_store<FAM, H, W, OBSK>(as, r, rows, s_obs);
    if (valid && j == 0) {
      as.reward[e] = r.reward;
      as.terminated[e] = r.term;
      as.truncated[e] = r.trunc;
    }
    acc.add(r);
    in.rec = r.nrec;
    in.episode = r.episode;
    in.balls = r.balls;
    dirty |= r.dirty;
  }
  if (valid) {
    if (j == 0) {
      a.agent[slot] = in.rec;
      a.episode[slot] = in.episode;
      if (FAM == FAM_DYNOBS) a.balls[slot] = in.balls;
    }
    if (dirty && j < H)
      a.grid[(tile * H + j) * TILE + st] = FAM == FAM_DYNOBS ? template_plane<FAM, H, W>(j) : rows[j * TILE];
  }
  acc.flush(a);
}

// f1: K consecutive steps of one tile in one CTA.  The grid rows
// stay in SMEM and the agent record, episode and balls in registers across
// the K steps; per step only the actions come in and obs / reward / flags go
// out (154 B per DoorKey env-step instead of 234).  Bit-identical to K
// navix_step calls; outputs of step t at [t][n].
template <int FAM, int H, int W, int OBSK>
__global__ void __launch_bounds__(TILE) navix_rollout_kernel(const KernelArgs a, int64_t K) {
  using C = Cfg<FAM, H, W>;
  auto& S = *reinterpret_cast<OneTileSmem<FAM, C::NPL, OBSK>*>(navix_dyn_smem);
  uint8_t* const s_obs = S.obs;
  auto& s_buf = S.buf;
  auto& s_scratch = S.scratch;
  auto& s_mbar = S.mbar;
  const int tid = threadIdx.x, le = 4 * (tid & 31) + (tid >> 5);
  const int64_t tile = blockIdx.x, tile0 = tile * TILE, slot = tile0 + tid, e = tile0 + le;
  const bool valid = e < a.n;
  const uint32_t mbar = smem_u32(&s_mbar);
  init_reset_queue_counter<FAM>();
  if (tid == 0) {
    mbar_init(mbar, 1);
    issue_tile_loads<FAM, H * C::RW, MODE_OBSERVE>(a, tile, s_buf, mbar);  // rows, agents (+ balls)
  }
  __syncthreads();
  mbar_wait(mbar, 0);
  EnvIn in{valid ? s_buf.agent[tid] : PADDING_AGENT_RECORD, 0u,
           FAM == FAM_DYNOBS && valid ? s_buf.balls[tid] : 0ull, a.episode[slot], true, false, true};
  bool dirty = false;
  StatsAcc acc;
  // actions from actions[t][n], or drawn in-kernel from the random-policy
  // stream (the one navix_sample_actions writes: bit-identical results)
  const bool draw = a.actions == nullptr;
  const uint32_t genv = a.env_begin + (uint32_t)e;
  auto policy = [&](int64_t t) -> uint32_t {
    const uint4 w = philox4x32_10(make_uint4(genv, a.act_t0 + (uint32_t)t, 2u << 16, 0u), a.act_key_lo, a.act_key_hi);
    return bounded(w.x, (uint32_t)C::NA);
  };
  uint32_t next_act = !valid ? 0u : draw ? policy(0) : a.actions[e];
  for (int64_t t = 0; t < K; ++t) {
    in.act = next_act;
    if (t + 1 < K && valid) next_act = draw ? policy(t + 1) : a.actions[(t + 1) * a.n + e];  // one step ahead
    KernelArgs as = a;
    as.obs = a.obs + t * a.n * obs_record_bytes(OBSK);
    as.reward = a.reward + t * a.n;
    as.terminated = a.terminated + t * a.n;
    as.truncated = a.truncated + t * a.n;
    as.bulk_obs = (reinterpret_cast<uintptr_t>(as.obs) & 15u) == 0;
    const EnvResult r = tile_compute<FAM, H, W, MODE_STEP, OBSK>(as, tile, &s_buf.rows[0][tid],
                                                           C::RW == 1 ? &s_scratch[0][tid] : nullptr, in,
                                                           s_obs, [&] {
      if (t > 0) {  // the previous step's store must have read s_obs
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
      }
    });
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    store_obs<OBSK>(as, tile, s_obs, tid, TILE, tid == 0);
    tile_store<FAM, MODE_STEP, false, false>(as, tile, r);
    acc.add(r);
    in.rec = r.nrec;
    in.episode = r.episode;
    in.balls = r.balls;
    in.tvalid = r.tvalid;
    dirty |= r.dirty;
  }
  if (valid) {
    a.agent[slot] = in.rec;
    a.episode[slot] = in.episode;
    if (FAM == FAM_DYNOBS) a.balls[slot] = in.balls;
  }
  if (dirty) {
    uint64_t* gdst = a.grid + tile0 * H * C::RW + tid;
#pragma unroll
    for (int p = 0; p < H * C::RW; ++p)
      gdst[p * TILE] = FAM == FAM_DYNOBS ? template_plane<FAM, H, W>(p) : s_buf.rows[p][tid];
  }
  acc.flush(a);
  if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// f3 (Table 5 `symbolic`): the full-grid encoding of MiniGrid's
// FullyObsWrapper — every cell (type, colour, state), the agent cell replaced
// by (10 agent, 0 red, dir); memory order [x][y][c] (R#32).  Not on the step
// path: one thread per env, staged in SMEM, coalesced copy-out.
template <int FAM, int H, int W, int OBSK>
__global__ void __launch_bounds__(TILE) full_obs_kernel(const KernelArgs a, uint8_t* out) {
  constexpr int CH = OBSK == OBS_CATEGORICAL ? 1 : 3;  // categorical: the entity type only (R#41)
  constexpr int PER = CH * W * H, RW = row_planes(W);
  constexpr bool STAGE = TILE * PER <= 32 * 1024;  // small grids: SMEM staging + coalesced copy-out
  __shared__ __align__(16) uint8_t s_out[STAGE ? TILE * PER : 16];
  const int tid = threadIdx.x, le = 4 * (tid & 31) + (tid >> 5);
  const int64_t tile0 = (int64_t)blockIdx.x * TILE, slot = tile0 + tid;
  const int64_t nv = a.n - tile0;
  const int nvalid = nv >= TILE ? TILE : (int)nv;
  const uint64_t rec = a.agent[slot];
  uint64_t pl[H * RW];
#pragma unroll
  for (int p = 0; p < H * RW; ++p) pl[p] = a.grid[tile0 * H * RW + p * TILE + tid];
  if (FAM == FAM_DYNOBS) {
    const uint64_t bl = a.balls[slot];
#pragma unroll
    for (int b = 0; b < Cfg<FAM, H, W>::NOBST; ++b) {
      const uint32_t q = (uint32_t)(bl >> (8 * b)) & 0xFF;
      const int bx = ball_x(W, q), by = ball_y(W, q);
#pragma unroll
      for (int p = 0; p < H * RW; ++p)
        if (q && p == by * RW + (bx >> 3))
          pl[p] = (pl[p] & ~(0xFFull << (8 * (bx & 7)))) | ((uint64_t)make_cell(K_BALL, COL_BLUE) << (8 * (bx & 7)));
    }
  }
  const int ax = (int)(rec & 0xFF), ay = (int)((rec >> 8) & 0xFF), dir = (int)((rec >> 16) & 3);
  uint8_t* o = STAGE ? s_out + le * PER : out + (tile0 + le) * PER;
  const bool write = STAGE || le < nvalid;
#pragma unroll
  for (int y = 0; y < H; ++y)
#pragma unroll
    for (int x = 0; x < W; ++x) {
      const uint32_t c = (uint32_t)(pl[y * RW + (x >> 3)] >> (8 * (x & 7))) & 0xFF, kind = c & 15;
      const bool ag = x == ax && y == ay;
      if (write) {
        uint8_t* t = o + (x * H + y) * CH;
        t[0] = ag ? 10 : (kind >= 11 ? 4 : kind);
        if (CH == 3) {
          t[1] = ag ? 0 : (c >> 4) & 7;
          t[2] = ag ? dir : (kind >= 11 ? kind - 10 : 0);
        }
      }
    }
  if (STAGE) {
    __syncthreads();
    uint8_t* dst = out + tile0 * PER;
    for (int i = tid; i < nvalid * PER; i += TILE) dst[i] = s_out[i];
  }
}

// ------------------------------------------------------------------ dispatch
// Experiment switches (A/B measurements only), read once per process.
inline int env_switch_onetile() {
  static const int v = [] { const char* e = getenv("NAVIX_STEP_KERNEL"); return e && e[0] == 'o' ? 1 : 0; }();
  return v;
}
inline int64_t env_switch_persist_ctas() {
  static const int64_t v = [] { const char* e = getenv("NAVIX_PERSIST_CTAS"); return e ? (int64_t)atoll(e) : (int64_t)0; }();
  return v;
}
inline int env_switch_pdl() {  // NAVIX_PDL=0: no PDL anywhere; =2: also on the small-batch step (A/B)
  static const int v = [] {
    const char* e = getenv("NAVIX_PDL");
    return e && e[0] == '0' ? 0 : e && e[0] == '2' ? 2 : 1;
  }();
  return v;
}

template <class K>
inline cudaError_t allow_dyn_smem(K kernel, size_t bytes) {
  return bytes > 48 * 1024
             ? cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes)
             : cudaSuccess;
}

// Per-device launch state of one kernel instantiation: the dynamic-SMEM
// opt-in (cudaFuncSetAttribute applies to the current device only), the SM
// count and the persistent kernel's occupancy.  Initialised once per device
// under std::call_once, so several devices (and threads) in one process each
// get their own.
constexpr int MAX_DEVICES = 64;
struct DeviceLaunchInfo {
  cudaError_t err = cudaSuccess;
  int n_sm = 0, per_sm = 0;
};

template <int FAM, int H, int W, int OBSK>
const DeviceLaunchInfo* device_launch_info() {
  using C = Cfg<FAM, H, W>;
  constexpr size_t DYN = sizeof(OneTileSmem<FAM, C::NPL, OBSK>);
  constexpr bool PERSIST = H * C::RW <= 16;
  constexpr size_t PDYN = sizeof(PersistSmem<FAM, C::NPL, OBSK>);
  static std::once_flag once[MAX_DEVICES];
  static DeviceLaunchInfo info[MAX_DEVICES];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) return nullptr;
  std::call_once(once[dev], [dev] {
    DeviceLaunchInfo& d = info[dev];
    cudaError_t e = cudaDeviceGetAttribute(&d.n_sm, cudaDevAttrMultiProcessorCount, dev);
    for (cudaError_t x : {allow_dyn_smem(navix_kernel<FAM, H, W, MODE_STEP, OBSK>, DYN),
                          allow_dyn_smem(navix_kernel<FAM, H, W, MODE_RESET, OBSK>, DYN),
                          allow_dyn_smem(navix_kernel<FAM, H, W, MODE_OBSERVE, OBSK>, DYN),
                          allow_dyn_smem(navix_rollout_kernel<FAM, H, W, OBSK>, DYN)})
      if (e == cudaSuccess) e = x;
    if constexpr (PERSIST) {
      if (e == cudaSuccess) e = allow_dyn_smem(navix_step_persistent<FAM, H, W, OBSK>, PDYN);
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&d.per_sm, navix_step_persistent<FAM, H, W, OBSK>, TILE,
                                                          PDYN);
    }
    if (d.per_sm < 1) d.per_sm = 1;
    d.err = e;
  });
  return &info[dev];
}

template <int FAM, int H, int W, int OBSK>
cudaError_t launch_fhwk(int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s) {
  const dim3 block(TILE);
  using C = Cfg<FAM, H, W>;
  constexpr size_t DYN = sizeof(OneTileSmem<FAM, C::NPL, OBSK>);
  const DeviceLaunchInfo* dl = device_launch_info<FAM, H, W, OBSK>();
  if (!dl) return cudaErrorInvalidDevice;
  if (dl->err != cudaSuccess) return dl->err;
  // the persistent kernel double-buffers the tile inputs in SMEM: grids up
  // to 16 row planes (8x8 and below, DistShift's 7 rows of 9); larger ones run
  // one tile per CTA, whose single buffer keeps more CTAs per SM (measured:
  // KeyCorridorS4R3 +24 %, SimpleCrossingS9N3 +11 % on the one-tile kernel)
  constexpr bool PERSIST = H * C::RW <= 16;
  constexpr size_t PDYN = sizeof(PersistSmem<FAM, C::NPL, OBSK>);
  // small batches: the multi-lane-per-env kernel (navix_step_wide)
  constexpr bool WIDE_OK = C::RW == 1 && FAM != FAM_GOTODOOR;
  if constexpr (WIDE_OK) {
    // KeyCorridor steps never take it: its level generator runs per lane
    // there (no warp-cooperative connect_all), and with steady-state resets
    // (episodes desynchronised) that lost at every size measured (512 envs
    // 13.2 us per step vs ~9.5 on the persistent kernel, 2,048: 19.1 vs 10.3)
    if (mode == MODE_STEP && FAM != FAM_KEYCORRIDOR && a.n <= a.wide_max) {
      // programmatic dependent launch only for grids of <= 48 CTAs (768
      // envs): there it hides the launch (2-8 %); on larger grids the next
      // step's CTAs, launched at once, sit on the SMs beside the running ones
      // and back-to-back steps ran 20-85 % slower from 1,536 envs on
      // (DESIGN.md §6.5); NAVIX_PDL=2 turns it on at every size (A/B)
      const unsigned wgrid = (unsigned)((a.n + WIDE_EPC - 1) / WIDE_EPC);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(wgrid);
      cfg.blockDim = block;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      const int pdl = env_switch_pdl();
      cfg.numAttrs = pdl == 2 || (pdl == 1 && wgrid <= 48u) ? 1 : 0;
      return cudaLaunchKernelEx(&cfg, navix_step_wide<FAM, H, W, OBSK>, a);
    }
  }
  if (mode == MODE_STEP && (env_switch_onetile() || !PERSIST)) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)n_tiles);
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = DYN;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, navix_kernel<FAM, H, W, MODE_STEP, OBSK>, a);
  } else if (mode == MODE_STEP) {
    if constexpr (PERSIST) {
      // persistent grid: as many CTAs as fit on this device at once
      int64_t cap = (int64_t)dl->per_sm * dl->n_sm;
      if (env_switch_persist_ctas() > 0) cap = env_switch_persist_ctas();
      const unsigned grid = (unsigned)(n_tiles < cap ? n_tiles : cap);
      // launched with programmatic stream serialization (PDL): back-to-back
      // steps overlap the launch of step t+1 with the tail of step t.  That
      // pays when the grid is full and the tiles fill its waves; when slots
      // stay free (fewer tiles than CTA slots, or a second wave less than
      // nine-tenths empty) the next step's CTAs launched into them slowed
      // the running ones: 8,192 - 131,072 envs 5-29 % faster without it,
      // 98,304 and >= 196,608 envs 1-5 % slower
      const bool pdl_pays = n_tiles >= cap && (n_tiles >= 2 * cap || 10 * (n_tiles - cap) < cap);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = block;
      cfg.dynamicSmemBytes = PDYN;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      const int pdl = env_switch_pdl();
      cfg.numAttrs = pdl == 2 || (pdl == 1 && pdl_pays) ? 1 : 0;
      return cudaLaunchKernelEx(&cfg, navix_step_persistent<FAM, H, W, OBSK>, a);
    }
  } else if (mode == MODE_OBS_TABLE) {
    if constexpr ((STATIC_LAYOUT<FAM> || LAYOUT_KEYED_VIS<FAM, W> || BORDER_OPACITY<FAM>) &&
                  OBSK == OBS_SYMBOLIC) {  // both kinds share it
      constexpr int NENT = vis_table_layouts<FAM, H, W>() * (W - 2) * (H - 2) * 4;
      obs_table_kernel<FAM, H, W><<<(NENT + TILE - 1) / TILE, block, 0, s>>>();
    }
  } else if (mode == MODE_FULL_OBS) {
    full_obs_kernel<FAM, H, W, OBSK><<<(unsigned)n_tiles, block, 0, s>>>(a, a.obs);
  } else if (mode == MODE_ROLLOUT) {
    if constexpr (WIDE_OK) {
      if (a.n <= a.wide_max_rollout) {
        navix_rollout_wide<FAM, H, W, OBSK><<<(unsigned)((a.n + WIDE_EPC - 1) / WIDE_EPC), block, 0, s>>>(
            a, a.rollout_steps);
        return cudaPeekAtLastError();
      }
    }
    navix_rollout_kernel<FAM, H, W, OBSK><<<(unsigned)n_tiles, block, DYN, s>>>(a, a.rollout_steps);
  } else if (mode == MODE_RESET) {
    navix_kernel<FAM, H, W, MODE_RESET, OBSK><<<(unsigned)n_tiles, block, DYN, s>>>(a);
  } else {
    navix_kernel<FAM, H, W, MODE_OBSERVE, OBSK><<<(unsigned)n_tiles, block, DYN, s>>>(a);
  }
  return cudaPeekAtLastError();
}

template <int FAM, int H, int W>
cudaError_t launch_fhw(int mode, const KernelArgs& a, int64_t n_tiles, cudaStream_t s) {
  return a.obs_kind == OBS_CATEGORICAL ? launch_fhwk<FAM, H, W, OBS_CATEGORICAL>(mode, a, n_tiles, s)
                                       : launch_fhwk<FAM, H, W, OBS_SYMBOLIC>(mode, a, n_tiles, s);
}

}  // namespace navix
