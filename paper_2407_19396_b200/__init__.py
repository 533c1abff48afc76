"""navix-b200: a B200-native batched MiniGrid step (NAVIX, arXiv 2407.19396).

The hot path is ``libnavix.so`` (sm_100a CUDA, C ABI in ``include/navix.h``);
``navix.NavixEnv`` is its thin torch/ctypes binding.
"""
from .navix import (  # noqa: F401
    EXPORTED_SYMBOLS,
    LIB_PATH,
    OBS_CATEGORICAL,
    OBS_SYMBOLIC,
    REWARD_MINIGRID,
    REWARD_NAVIX,
    STATS_FIELDS,
    build_id,
    NavixEnv,
    NavixError,
    load_library,
    shard_range,
    spec_of,
    state_bytes,
)
