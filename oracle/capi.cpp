// oracle/capi.cpp — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
//
// extern "C" entry points of liboracle.so, loaded by oracle/binding.py for
// tests/, __graft_entry__.smoke() and bench.py's CPU baseline.  A handle holds
// n_local independent environments with global indices
// [env_begin, env_begin + n_local) of a batch of n_total (shard semantics of
// the product ABI), stepped one after another on one host thread.
#include <cstring>
#include <string>
#include <vector>

#include "oracle.hpp"

using namespace oracle;

namespace {
struct Handle {
  Spec spec;
  std::vector<Env> envs;
};
}  // namespace

extern "C" {

// out[0..7] = height, width, max_steps, n_actions, family, obs_bytes (147),
//             export_bytes_per_env, n_obstacles.  Returns 0 if unknown.
int oracle_spec(const char* env_id, int32_t* out) {
  Spec s;
  if (!parse_env_id(env_id, &s)) return 0;
  out[0] = s.height; out[1] = s.width; out[2] = s.max_steps; out[3] = s.n_actions;
  out[4] = s.family; out[5] = 147; out[6] = export_bytes_per_env(s); out[7] = s.n_obstacles;
  return 1;
}

void* oracle_create(const char* env_id, int64_t n_total, int64_t env_begin, int64_t n_local,
                    uint64_t seed, int reward_mode) {
  Spec s;
  if (!parse_env_id(env_id, &s)) return nullptr;
  if (n_local <= 0 || env_begin < 0 || env_begin + n_local > n_total) return nullptr;
  Handle* h = new Handle;
  h->spec = s;
  h->envs.resize((size_t)n_local);
  for (int64_t i = 0; i < n_local; ++i) {
    Env& e = h->envs[(size_t)i];
    e.spec = s;
    e.reward_mode = reward_mode;
    e.seed = seed;
    e.global_index = (uint32_t)(env_begin + i);
  }
  return h;
}

void oracle_destroy(void* hp) { delete (Handle*)hp; }

// reset(key): episode 0 for every env; statistics zeroed.
void oracle_reset(void* hp, uint8_t* obs) {
  Handle* h = (Handle*)hp;
  for (size_t i = 0; i < h->envs.size(); ++i) {
    Env& e = h->envs[i];
    for (auto& v : e.stats) v = 0;
    e.episode = 0;
    e.generate();
    if (obs) e.gen_obs(obs + i * 147);
  }
}

// step(timestep, action) (Code 1 P:264) for every env.
void oracle_step(void* hp, const uint8_t* actions, uint8_t* obs, float* reward, uint8_t* term,
                 uint8_t* trunc) {
  Handle* h = (Handle*)hp;
  for (size_t i = 0; i < h->envs.size(); ++i) {
    Env& e = h->envs[i];
    StepOut o = e.step((int)actions[i]);
    if (obs) e.gen_obs(obs + i * 147);
    if (reward) reward[i] = o.reward;
    if (term) term[i] = o.terminated ? 1 : 0;
    if (trunc) trunc[i] = o.truncated ? 1 : 0;
  }
}

void oracle_observe(void* hp, uint8_t* obs) {
  Handle* h = (Handle*)hp;
  for (size_t i = 0; i < h->envs.size(); ++i) h->envs[i].gen_obs(obs + i * 147);
}

void oracle_set_event_functions(void* hp, uint32_t reward_events, uint32_t termination_events) {
  Handle* h = (Handle*)hp;
  for (auto& e : h->envs) { e.reward_events = reward_events; e.termination_events = termination_events; }
}

void oracle_set_reward_costs(void* hp, float time_cost, float action_cost) {
  Handle* h = (Handle*)hp;
  for (auto& e : h->envs) { e.time_cost = time_cost; e.action_cost = action_cost; }
}

// out[i] = uint8[width][height][3] full-grid symbolic observation of env i.
void oracle_observe_full(void* hp, uint8_t* out) {
  Handle* h = (Handle*)hp;
  const size_t per = (size_t)h->spec.width * h->spec.height * 3;
  for (size_t i = 0; i < h->envs.size(); ++i) h->envs[i].gen_full_obs(out + i * per);
}

int64_t oracle_export(void* hp, uint8_t* buf, int64_t cap) {
  Handle* h = (Handle*)hp;
  int64_t per = export_bytes_per_env(h->spec);
  int64_t need = per * (int64_t)h->envs.size();
  if (!buf) return need;
  if (cap < need) return -1;
  for (size_t i = 0; i < h->envs.size(); ++i) export_env(h->envs[i], buf + i * per);
  return need;
}

// Returns the index of the first env whose record is rejected, or -1 if all ok.
int64_t oracle_import(void* hp, const uint8_t* buf, int64_t n) {
  Handle* h = (Handle*)hp;
  int64_t per = export_bytes_per_env(h->spec);
  if (n != per * (int64_t)h->envs.size()) return 0;
  for (size_t i = 0; i < h->envs.size(); ++i)
    if (!import_env(h->envs[i], buf + i * per)) return (int64_t)i;
  return -1;
}

// int64[8]: episodes, sum_len, n_success, sum_success_step, n_lava,
// n_collision, n_truncated, gen_failures.
void oracle_stats(void* hp, int64_t* out) {
  Handle* h = (Handle*)hp;
  for (int k = 0; k < 8; ++k) out[k] = 0;
  for (auto& e : h->envs)
    for (int k = 0; k < 8; ++k) out[k] += e.stats[k];
}

void oracle_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  philox4x32_10(ctr, key, out);
}

// Random-policy action stream: a[t][env] =
// bounded(word0(Philox(ctr=(env, t, 2<<16, 0), key=action_seed)), n_actions).
void oracle_sample_actions(uint64_t action_seed, int64_t env_begin, int64_t n, int64_t t0,
                           int64_t steps, int n_actions, uint8_t* out) {
  uint32_t key[2] = {(uint32_t)(action_seed & 0xffffffffu), (uint32_t)(action_seed >> 32)};
  for (int64_t t = 0; t < steps; ++t)
    for (int64_t i = 0; i < n; ++i) {
      uint32_t ctr[4] = {(uint32_t)(env_begin + i), (uint32_t)(t0 + t), 2u << 16, 0u};
      uint32_t w[4];
      philox4x32_10(ctr, key, w);
      out[t * n + i] = (uint8_t)bounded(w[0], (uint32_t)n_actions);
    }
}

// Literal [MG] process_vis on a 7x7 view whose cell (i, j) is a Wall when
// opaque[i*7+j] != 0 and None otherwise; agent at (3, 6).  mask[i*7+j].
void oracle_process_vis7(const uint8_t* opaque, uint8_t* mask) {
  Grid g(7, 7);
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j)
      if (opaque[i * 7 + j]) g.set(i, j, make_wall());
  std::vector<uint8_t> m = g.process_vis(3, 6);
  for (int k = 0; k < 49; ++k) mask[k] = m[k];
}

// Slice + rotate_left^(dir+1) (the [MG] view transform) applied to a W x H
// grid whose cell (x, y) carries tag y*W+x; out_tag[i*7+j] = the tag landing
// in view cell (i, j), or -1 for an out-of-grid (Wall-filled) cell.
void oracle_view_tags(int W, int H, int ax, int ay, int dir, int32_t* out_tag) {
  Env e;
  e.grid = Grid(W, H);
  for (int y = 0; y < H; ++y)
    for (int x = 0; x < W; ++x) {
      Obj o = make_key(0);
      o.tag = y * W + x + 1;
      e.grid.set(x, y, o);
    }
  const int R = 7;
  int topX, topY;
  if (dir == 0) { topX = ax; topY = ay - R / 2; }
  else if (dir == 1) { topX = ax - R / 2; topY = ay; }
  else if (dir == 2) { topX = ax - R + 1; topY = ay - R / 2; }
  else { topX = ax - R / 2; topY = ay - R + 1; }
  Grid g = e.grid.slice(topX, topY, R, R);
  for (int i = 0; i < dir + 1; ++i) g = g.rotate_left();
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) {
      const Cell& c = g.get(i, j);
      out_tag[i * 7 + j] = (c && c->type == T_KEY) ? c->tag - 1 : -1;
    }
}

// Success reward (Eq. 1 / P:223) exposed for the reward pins (P4).
float oracle_success_reward(int mode, int sc, int T) { return success_reward(mode, sc, T); }

}  // extern "C"
