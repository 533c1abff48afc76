"""Thin Python binding of libnavix.so (include/navix.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module
only checks tensor shapes/devices and passes raw pointers plus the current
torch CUDA stream.  There is no CPU fallback: constructing an env without the
built library or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# NAVIX_LIBRARY: another build of the same ABI, for A/B measurements only (the
# tests assert the default in-tree library matches the source tree)
LIB_PATH = os.environ.get("NAVIX_LIBRARY") or os.path.join(_HERE, "libnavix.so")
_lib = None

NAVIX_OK, NAVIX_E_UNKNOWN_ENV, NAVIX_E_INVALID_ARG, NAVIX_E_CUDA, NAVIX_E_NOMEM, NAVIX_E_UNSUPPORTED = range(6)
REWARD_MINIGRID, REWARD_NAVIX = 0, 1
# observation kinds (Table 5; include/navix.h NAVIX_OBS_*)
OBS_SYMBOLIC, OBS_CATEGORICAL = 0, 1
_OBS_KINDS = {"symbolic": OBS_SYMBOLIC, "categorical": OBS_CATEGORICAL}
STATS_FIELDS = ("episodes", "sum_len", "n_success", "sum_success_step",
                "n_lava", "n_failure", "n_truncated", "gen_failures")
EXPORTED_SYMBOLS = (
    "navix_spec_of", "navix_state_bytes", "navix_create", "navix_create_shard", "navix_reset",
    "navix_step", "navix_rollout", "navix_observe", "navix_observe_full", "navix_set_reward_costs", "navix_set_observation",
    "navix_set_event_functions", "navix_rollout_random", "navix_reset_seed", "navix_observe_mission", "navix_sample_actions", "navix_step_host", "navix_stats",
    "navix_state_export", "navix_state_import", "navix_info", "navix_destroy", "navix_last_error", "navix_build_id", "navix_set_small_batch_threshold",
)


class NavixError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"navix status {status}: {msg}")
        self.status = status


class _Spec(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "height", "width", "view", "n_actions", "max_steps", "obs_bytes", "family", "n_obstacles",
        "export_bytes")]


@dataclass(frozen=True)
class Spec:
    height: int
    width: int
    view: int
    n_actions: int
    max_steps: int
    obs_bytes: int
    family: int
    n_obstacles: int
    export_bytes: int


def load_library():
    """Load libnavix.so from the package directory (build it with build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2407_19396_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I64, U64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_size_t
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "navix_spec_of": ([ctypes.c_char_p, ctypes.POINTER(_Spec)], I32),
        "navix_state_bytes": ([ctypes.c_char_p, I64], SZ),
        "navix_create": ([ctypes.c_char_p, I64, U64, PP], I32),
        "navix_create_shard": ([ctypes.c_char_p, I64, I64, I64, U64, I32, P, I32, PP], I32),
        "navix_reset": ([P, P, P], I32),
        "navix_reset_seed": ([P, U64, P, P], I32),
        "navix_step": ([P, P, P, P, P, P, P], I32),
        "navix_observe": ([P, P, P], I32),
        "navix_rollout": ([P, P, I64, P, P, P, P, P], I32),
        "navix_rollout_random": ([P, U64, I64, I64, P, P, P, P, P], I32),
        "navix_observe_full": ([P, P, P], I32),
        "navix_observe_mission": ([P, P, P], I32),
        "navix_set_reward_costs": ([P, ctypes.c_float, ctypes.c_float], I32),
        "navix_set_observation": ([P, I32], I32),
        "navix_set_event_functions": ([P, ctypes.c_uint32, ctypes.c_uint32], I32),
        "navix_sample_actions": ([P, U64, I64, I64, P, P], I32),
        "navix_step_host": ([P, P, P, P, P, P, P], I32),
        "navix_stats": ([P, P, P], I32),
        "navix_state_export": ([P, P, SZ, ctypes.POINTER(SZ)], I32),
        "navix_state_import": ([P, P, SZ], I32),
        "navix_info": ([P, P], I32),
        "navix_destroy": ([P], None),
        "navix_last_error": ([], ctypes.c_char_p),
        "navix_build_id": ([], ctypes.c_char_p),
        "navix_set_small_batch_threshold": ([P, I64], I32),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("NAVIX_LIBRARY") and not hasattr(lib, name):
            continue  # A/B against an older build: its missing entry points stay unbound
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def build_id() -> str:
    """Source hash libnavix.so was compiled from (see build.source_hash)."""
    return load_library().navix_build_id().decode()


def _check(status: int):
    if status != NAVIX_OK:
        raise NavixError(status, load_library().navix_last_error().decode())


def spec_of(env_id: str) -> Spec:
    s = _Spec()
    st = load_library().navix_spec_of(env_id.encode(), ctypes.byref(s))
    if st not in (NAVIX_OK, NAVIX_E_UNSUPPORTED):
        _check(st)
    return Spec(*[getattr(s, f) for f, _ in _Spec._fields_])


def state_bytes(env_id: str, num_envs: int) -> int:
    return int(load_library().navix_state_bytes(env_id.encode(), num_envs))


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class NavixEnv:
    """A batch (or one shard of a batch) of MiniGrid environments on one GPU.

    ``reset()`` / ``step(actions)`` return CUDA tensors written by the kernels:
    obs uint8[n, 7, 7, 3] ([vi][vj][channel]), reward float32[n],
    terminated / truncated bool-valued uint8[n].  Output tensors are reused
    between calls unless ``out=`` is given.  ``observation="categorical"``
    (Table 5 categorical / categorical_first_person) makes every obs output
    the entity type alone: uint8[n, 7, 7] and uint8[n, width, height].
    """

    def __init__(self, env_id: str, num_envs: int, seed: int = 0, *, device=None,
                 reward_mode: int = REWARD_MINIGRID, env_begin: int = 0,
                 num_envs_total: int | None = None, state: torch.Tensor | None = None,
                 observation: str = "symbolic"):
        if not torch.cuda.is_available():
            raise RuntimeError("NavixEnv needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.env_id = env_id
        self.spec = spec_of(env_id)
        self.n = int(num_envs)
        self.env_begin = int(env_begin)
        self.n_total = self.env_begin + self.n if num_envs_total is None else int(num_envs_total)
        self.seed = int(seed)
        if state is not None:
            need = state_bytes(env_id, self.n)
            if (state.device != self.device or state.dtype != torch.uint8 or not state.is_contiguous()
                    or state.numel() < need or state.data_ptr() % 256):
                raise ValueError(f"state must be a contiguous, 256-byte aligned uint8 tensor of >= {need} bytes "
                                 f"on {self.device}")
        self._state = state
        h = ctypes.c_void_p()
        _check(self.lib.navix_create_shard(
            env_id.encode(), self.n_total, self.env_begin, self.n, self.seed & (2 ** 64 - 1),
            self.device.index, None if state is None else _ptr(state), reward_mode, ctypes.byref(h)))
        self.h = h
        if observation not in _OBS_KINDS:
            raise ValueError(f"observation must be one of {sorted(_OBS_KINDS)}")
        self.observation = observation
        _check(self.lib.navix_set_observation(self.h, _OBS_KINDS[observation]))
        self.obs_shape = (7, 7, 3) if observation == "symbolic" else (7, 7)
        s = self.spec
        self.full_shape = (s.width, s.height, 3) if observation == "symbolic" else (s.width, s.height)
        dev = self.device
        self.obs = torch.empty((self.n, *self.obs_shape), dtype=torch.uint8, device=dev)
        self.reward = torch.empty(self.n, dtype=torch.float32, device=dev)
        self.terminated = torch.empty(self.n, dtype=torch.uint8, device=dev)
        self.truncated = torch.empty(self.n, dtype=torch.uint8, device=dev)
        self._stats = torch.zeros(8, dtype=torch.int64, device=dev)

    def close(self):
        if getattr(self, "h", None):
            self.lib.navix_destroy(self.h)
            self.h = None

    __del__ = close

    def _check_out(self, t: torch.Tensor, shape, dtype):
        if t.device != self.device or t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
            raise ValueError(f"expected contiguous {dtype} {tuple(shape)} on {self.device}, got "
                             f"{t.dtype} {tuple(t.shape)} on {t.device}")

    def reset(self, out: torch.Tensor | None = None) -> torch.Tensor:
        obs = self.obs if out is None else out
        self._check_out(obs, (self.n, *self.obs_shape), torch.uint8)
        _check(self.lib.navix_reset(self.h, _ptr(obs), _stream(self.device)))
        return obs

    def reset_seed(self, seed: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """reset(key) with a new key: every later level uses Philox key `seed`.
        Captured CUDA graphs keep the old key: recapture them after this call."""
        obs = self.obs if out is None else out
        self._check_out(obs, (self.n, *self.obs_shape), torch.uint8)
        self.seed = int(seed)
        _check(self.lib.navix_reset_seed(self.h, self.seed & (2 ** 64 - 1), _ptr(obs), _stream(self.device)))
        return obs

    def step(self, actions: torch.Tensor, out=None):
        self._check_out(actions, (self.n,), torch.uint8)
        obs, rew, term, trunc = out if out is not None else (
            self.obs, self.reward, self.terminated, self.truncated)
        self._check_out(obs, (self.n, *self.obs_shape), torch.uint8)
        self._check_out(rew, (self.n,), torch.float32)
        self._check_out(term, (self.n,), torch.uint8)
        self._check_out(trunc, (self.n,), torch.uint8)
        _check(self.lib.navix_step(self.h, _ptr(actions), _ptr(obs), _ptr(rew), _ptr(term), _ptr(trunc),
                                   _stream(self.device)))
        return obs, rew, term, trunc

    def rollout(self, actions: torch.Tensor, out=None):
        """K steps in one launch (state on chip): actions uint8[K, n] ->
        obs uint8[K, n, 7, 7, 3], reward float32[K, n], terminated / truncated uint8[K, n]."""
        if actions.dim() != 2:
            raise ValueError("actions must be uint8[K, n]")
        K = actions.shape[0]
        self._check_out(actions, (K, self.n), torch.uint8)
        dev = self.device
        if out is None:
            out = (torch.empty((K, self.n, *self.obs_shape), dtype=torch.uint8, device=dev),
                   torch.empty((K, self.n), dtype=torch.float32, device=dev),
                   torch.empty((K, self.n), dtype=torch.uint8, device=dev),
                   torch.empty((K, self.n), dtype=torch.uint8, device=dev))
        obs, rew, term, trunc = out
        self._check_out(obs, (K, self.n, *self.obs_shape), torch.uint8)
        self._check_out(rew, (K, self.n), torch.float32)
        self._check_out(term, (K, self.n), torch.uint8)
        self._check_out(trunc, (K, self.n), torch.uint8)
        _check(self.lib.navix_rollout(self.h, _ptr(actions), K, _ptr(obs), _ptr(rew), _ptr(term), _ptr(trunc),
                                      _stream(dev)))
        return obs, rew, term, trunc

    def rollout_random(self, action_seed: int, t0: int, steps: int, out=None):
        """K steps in one launch under the in-kernel uniform random policy
        (the sample_actions(action_seed, t0, K) stream); outputs as rollout()."""
        K = int(steps)
        dev = self.device
        if out is None:
            out = (torch.empty((K, self.n, *self.obs_shape), dtype=torch.uint8, device=dev),
                   torch.empty((K, self.n), dtype=torch.float32, device=dev),
                   torch.empty((K, self.n), dtype=torch.uint8, device=dev),
                   torch.empty((K, self.n), dtype=torch.uint8, device=dev))
        obs, rew, term, trunc = out
        self._check_out(obs, (K, self.n, *self.obs_shape), torch.uint8)
        self._check_out(rew, (K, self.n), torch.float32)
        self._check_out(term, (K, self.n), torch.uint8)
        self._check_out(trunc, (K, self.n), torch.uint8)
        _check(self.lib.navix_rollout_random(self.h, action_seed & (2 ** 64 - 1), t0, K, _ptr(obs), _ptr(rew),
                                             _ptr(term), _ptr(trunc), _stream(dev)))
        return obs, rew, term, trunc

    def set_reward_costs(self, time_cost: float = 0.0, action_cost: float = 0.0) -> None:
        """Compose -time_cost per step and -action_cost per non-done action (Table 6).
        Captured CUDA graphs keep the old costs: recapture them after this call."""
        _check(self.lib.navix_set_reward_costs(self.h, time_cost, action_cost))

    def set_small_batch_threshold(self, max_envs: int) -> None:
        """Steps of at most max_envs envs use the multi-lane-per-env kernel (0: never).
        Bit-identical results; captured CUDA graphs keep the old choice."""
        _check(self.lib.navix_set_small_batch_threshold(self.h, int(max_envs)))

    def set_event_functions(self, reward_events: int = 7, termination_events: int = 7) -> None:
        """Table 6 / 7 selection: bit 0 goal/success, 1 lava, 2 failure; 0 = `free`.
        Captured CUDA graphs keep the old selection: recapture them after this call."""
        _check(self.lib.navix_set_event_functions(self.h, reward_events, termination_events))

    def observe_full(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """Table 5 `symbolic`: uint8[n, width, height, 3], agent cell (10, 0, dir)
        (`categorical`: uint8[n, width, height], agent 10)."""
        o = torch.empty((self.n, *self.full_shape), dtype=torch.uint8, device=self.device) if out is None else out
        self._check_out(o, (self.n, *self.full_shape), torch.uint8)
        _check(self.lib.navix_observe_full(self.h, _ptr(o), _stream(self.device)))
        return o

    def observe_mission(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """GoToDoor: uint8[n] colour index of each env's target door (the mission)."""
        o = torch.empty(self.n, dtype=torch.uint8, device=self.device) if out is None else out
        self._check_out(o, (self.n,), torch.uint8)
        _check(self.lib.navix_observe_mission(self.h, _ptr(o), _stream(self.device)))
        return o

    def observe(self, out: torch.Tensor | None = None) -> torch.Tensor:
        obs = self.obs if out is None else out
        self._check_out(obs, (self.n, *self.obs_shape), torch.uint8)
        _check(self.lib.navix_observe(self.h, _ptr(obs), _stream(self.device)))
        return obs

    def sample_actions(self, action_seed: int, t0: int, steps: int, out: torch.Tensor | None = None):
        a = torch.empty((steps, self.n), dtype=torch.uint8, device=self.device) if out is None else out
        self._check_out(a, (steps, self.n), torch.uint8)
        _check(self.lib.navix_sample_actions(self.h, action_seed & (2 ** 64 - 1), t0, steps, _ptr(a),
                                             _stream(self.device)))
        return a

    def step_host(self, actions: torch.Tensor, obs: torch.Tensor, reward: torch.Tensor,
                  terminated: torch.Tensor, truncated: torch.Tensor):
        """End-to-end step on HOST tensors (pinned preferred); synchronises."""
        for t, shape, dt in ((actions, (self.n,), torch.uint8), (obs, (self.n, *self.obs_shape), torch.uint8),
                             (reward, (self.n,), torch.float32), (terminated, (self.n,), torch.uint8),
                             (truncated, (self.n,), torch.uint8)):
            if t.device.type != "cpu" or t.dtype != dt or tuple(t.shape) != shape or not t.is_contiguous():
                raise ValueError("step_host expects contiguous host tensors")
        _check(self.lib.navix_step_host(self.h, _ptr(actions), _ptr(obs), _ptr(reward), _ptr(terminated),
                                        _ptr(truncated), _stream(self.device)))

    def stats(self, out: torch.Tensor | None = None) -> torch.Tensor:
        """Device int64[8] episode statistics of this shard (see STATS_FIELDS)."""
        o = self._stats if out is None else out
        self._check_out(o, (8,), torch.int64)
        _check(self.lib.navix_stats(self.h, _ptr(o), _stream(self.device)))
        return o

    def export_state(self) -> np.ndarray:
        per = self.spec.export_bytes
        buf = np.zeros(self.n * per, np.uint8)
        written = ctypes.c_size_t()
        _check(self.lib.navix_state_export(self.h, buf.ctypes.data_as(ctypes.c_void_p), buf.size,
                                           ctypes.byref(written)))
        assert written.value == buf.size
        return buf.reshape(self.n, per)

    def import_state(self, records: np.ndarray) -> None:
        r = np.ascontiguousarray(records, np.uint8).reshape(-1)
        _check(self.lib.navix_state_import(self.h, r.ctypes.data_as(ctypes.c_void_p), r.size))


def shard_range(num_envs_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous global env range [begin, end) of `rank`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    begin = rank * num_envs_total // world
    end = (rank + 1) * num_envs_total // world
    return begin, end
