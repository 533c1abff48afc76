"""CPU oracle of the batched MiniGrid step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline
(``cpu_baseline`` and ``--impl reference``) may import this package.  The
product package ``paper_2407_19396_b200`` never imports it and shares no code
with it.  See ``oracle/oracle.hpp`` for the citation conventions.
"""
from .binding import (  # noqa: F401
    OracleEnv,
    build_oracle,
    oracle_lib,
    philox4x32_10,
    process_vis7,
    sample_actions,
    spec_of,
    success_reward,
    view_tags,
)
