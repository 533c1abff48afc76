"""ctypes binding of liboracle.so — TEST INFRASTRUCTURE ONLY (see __init__)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRCS = ["minigrid.cpp", "levels.cpp", "capi.cpp"]
_lib = None

STATS_FIELDS = (
    "episodes", "sum_len", "n_success", "sum_success_step",
    "n_lava", "n_failure", "n_truncated", "gen_failures",
)


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2 -ffp-contract=off: no FMA contraction, R#2)."""
    srcs = [os.path.join(_HERE, s) for s in _SRCS]
    hdr = os.path.join(_HERE, "oracle.hpp")
    if not force and os.path.exists(_SO):
        newest = max(os.path.getmtime(p) for p in srcs + [hdr])
        if os.path.getmtime(_SO) >= newest:
            return _SO
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
           *srcs, "-o", _SO]
    subprocess.run(cmd, check=True)
    return _SO


def oracle_lib():
    global _lib
    if _lib is not None:
        return _lib
    build_oracle()
    lib = ctypes.CDLL(_SO)
    P, I64, U64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
    lib.oracle_spec.argtypes = [ctypes.c_char_p, P]
    lib.oracle_spec.restype = I32
    lib.oracle_create.argtypes = [ctypes.c_char_p, I64, I64, I64, U64, I32]
    lib.oracle_create.restype = P
    lib.oracle_destroy.argtypes = [P]
    lib.oracle_reset.argtypes = [P, P]
    lib.oracle_step.argtypes = [P, P, P, P, P, P]
    lib.oracle_observe.argtypes = [P, P]
    lib.oracle_export.argtypes = [P, P, I64]
    lib.oracle_export.restype = I64
    lib.oracle_import.argtypes = [P, P, I64]
    lib.oracle_import.restype = I64
    lib.oracle_stats.argtypes = [P, P]
    lib.oracle_philox4x32_10.argtypes = [P, P, P]
    lib.oracle_sample_actions.argtypes = [U64, I64, I64, I64, I64, I32, P]
    lib.oracle_process_vis7.argtypes = [P, P]
    lib.oracle_view_tags.argtypes = [I32, I32, I32, I32, I32, P]
    lib.oracle_set_reward_costs.argtypes = [P, ctypes.c_float, ctypes.c_float]
    lib.oracle_set_event_functions.argtypes = [P, ctypes.c_uint32, ctypes.c_uint32]
    lib.oracle_observe_full.argtypes = [P, P]
    lib.oracle_success_reward.argtypes = [I32, I32, I32]
    lib.oracle_success_reward.restype = ctypes.c_float
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class OracleSpec:
    height: int
    width: int
    max_steps: int
    n_actions: int
    family: int
    obs_bytes: int
    export_bytes: int
    n_obstacles: int


def spec_of(env_id: str) -> OracleSpec:
    out = np.zeros(8, np.int32)
    if not oracle_lib().oracle_spec(env_id.encode(), _ptr(out)):
        raise KeyError(f"oracle: unknown env id {env_id!r}")
    return OracleSpec(*[int(v) for v in out])


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, np.uint32).copy()
    k = np.asarray(key, np.uint32).copy()
    o = np.zeros(4, np.uint32)
    oracle_lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def sample_actions(action_seed: int, env_begin: int, n: int, t0: int, steps: int,
                   n_actions: int) -> np.ndarray:
    out = np.zeros((steps, n), np.uint8)
    oracle_lib().oracle_sample_actions(action_seed, env_begin, n, t0, steps, n_actions, _ptr(out))
    return out


def process_vis7(opaque: np.ndarray) -> np.ndarray:
    """opaque[i, j] (7x7, i lateral, j row) -> literal [MG] process_vis mask[i, j]."""
    o = np.ascontiguousarray(opaque, np.uint8).reshape(49)
    m = np.zeros(49, np.uint8)
    oracle_lib().oracle_process_vis7(_ptr(o), _ptr(m))
    return m.reshape(7, 7)


def view_tags(W: int, H: int, ax: int, ay: int, d: int) -> np.ndarray:
    out = np.zeros(49, np.int32)
    oracle_lib().oracle_view_tags(W, H, ax, ay, d, _ptr(out))
    return out.reshape(7, 7)


def success_reward(mode: int, sc: int, T: int) -> float:
    return float(oracle_lib().oracle_success_reward(mode, sc, T))


class OracleEnv:
    """n_local MiniGrid environments (global indices env_begin..) on one host thread."""

    def __init__(self, env_id: str, num_envs: int, seed: int = 0, *, reward_mode: int = 0,
                 env_begin: int = 0, num_envs_total: int | None = None):
        self.lib = oracle_lib()
        self.spec = spec_of(env_id)
        self.env_id = env_id
        self.n = int(num_envs)
        total = self.n + env_begin if num_envs_total is None else int(num_envs_total)
        self.h = self.lib.oracle_create(env_id.encode(), total, env_begin, self.n, seed, reward_mode)
        if not self.h:
            raise ValueError("oracle_create rejected its arguments")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.oracle_destroy(h)
            self.h = None

    def reset(self) -> np.ndarray:
        obs = np.zeros((self.n, 7, 7, 3), np.uint8)
        self.lib.oracle_reset(self.h, _ptr(obs))
        return obs

    def step(self, actions):
        a = np.ascontiguousarray(actions, np.uint8)
        assert a.shape == (self.n,)
        obs = np.zeros((self.n, 7, 7, 3), np.uint8)
        rew = np.zeros(self.n, np.float32)
        term = np.zeros(self.n, np.uint8)
        trunc = np.zeros(self.n, np.uint8)
        self.lib.oracle_step(self.h, _ptr(a), _ptr(obs), _ptr(rew), _ptr(term), _ptr(trunc))
        return obs, rew, term, trunc

    def step_no_obs(self, actions):
        a = np.ascontiguousarray(actions, np.uint8)
        rew = np.zeros(self.n, np.float32)
        term = np.zeros(self.n, np.uint8)
        trunc = np.zeros(self.n, np.uint8)
        self.lib.oracle_step(self.h, _ptr(a), None, _ptr(rew), _ptr(term), _ptr(trunc))
        return rew, term, trunc

    def observe(self) -> np.ndarray:
        obs = np.zeros((self.n, 7, 7, 3), np.uint8)
        self.lib.oracle_observe(self.h, _ptr(obs))
        return obs

    def set_reward_costs(self, time_cost: float, action_cost: float) -> None:
        self.lib.oracle_set_reward_costs(self.h, time_cost, action_cost)

    def set_event_functions(self, reward_events: int, termination_events: int) -> None:
        self.lib.oracle_set_event_functions(self.h, reward_events, termination_events)

    def observe_full(self) -> np.ndarray:
        s = self.spec
        out = np.zeros((self.n, s.width, s.height, 3), np.uint8)
        self.lib.oracle_observe_full(self.h, _ptr(out))
        return out

    def export(self) -> np.ndarray:
        buf = np.zeros(self.n * self.spec.export_bytes, np.uint8)
        got = self.lib.oracle_export(self.h, _ptr(buf), buf.size)
        assert got == buf.size
        return buf.reshape(self.n, self.spec.export_bytes)

    def import_(self, records: np.ndarray) -> None:
        r = np.ascontiguousarray(records, np.uint8).reshape(-1)
        bad = self.lib.oracle_import(self.h, _ptr(r), r.size)
        if bad != -1:
            raise ValueError(f"oracle_import rejected env record {bad}")

    def stats(self) -> np.ndarray:
        out = np.zeros(8, np.int64)
        self.lib.oracle_stats(self.h, _ptr(out))
        return out
