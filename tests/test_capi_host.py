"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/navix.h declares, parses Table 9 ids, sizes state, and
rejects bad arguments with a status and a message."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_are_exported():
    from paper_2407_19396_b200 import EXPORTED_SYMBOLS, load_library
    hdr = open(os.path.join(ROOT, "include", "navix.h")).read()
    declared = set(re.findall(r"NAVIX_API\s+[\w\s\*]+?\b(navix_\w+)\s*\(", hdr))
    assert declared == set(EXPORTED_SYMBOLS)
    lib = load_library()
    for name in declared:
        assert hasattr(lib, name), name


@pytest.mark.parametrize("env_id,h,w,T,na,fam", [
    ("Navix-Empty-5x5-v0", 5, 5, 100, 7, 0),
    ("MiniGrid-Empty-8x8-v0", 8, 8, 256, 7, 0),
    ("DoorKey-8x8", 8, 8, 640, 7, 1),
    ("Navix-Dynamic-Obstacles-8x8-v0", 8, 8, 256, 3, 2),
    ("Navix-KeyCorridorS3R3-v0", 7, 7, 270, 7, 3),
    ("KeyCorridorS3R1", 3, 7, 270, 7, 3),
    ("Navix-LavaGapS7-v0", 7, 7, 196, 7, 4),
    ("Navix-Empty-Random-6x6", 6, 6, 144, 7, 5),
    ("Navix-DistShift1-v0", 7, 9, 252, 7, 6),
    ("Navix-DistShift2-v0", 7, 9, 252, 7, 6),
    ("Navix-SimpleCrossingS9N2-v0", 9, 9, 324, 7, 7),
    ("Navix-Crossings-S11N5-v0", 11, 11, 484, 7, 7),
    ("Navix-Crossings-S9N1-v0", 9, 9, 324, 7, 7),
    ("MiniGrid-LavaCrossingS9N2-v0", 9, 9, 324, 7, 7),
    ("Navix-LavaGap-S7-v0", 7, 7, 196, 7, 4),
    ("Navix-LavaGap-S5-v0", 5, 5, 100, 7, 4),
    ("Navix-DoorKey-Random-5x5", 5, 5, 250, 7, 1),
    ("Navix-GoToDoor-8x8-v0", 8, 8, 256, 7, 8),
    ("Navix-FourRooms-v0", 17, 17, 100, 7, 9),
    ("MiniGrid-Dynamic-Obstacles-Random-6x6-v0", 6, 6, 144, 3, 2),
])
def test_spec_of_table9_ids(env_id, h, w, T, na, fam):
    from oracle import spec_of as oracle_spec
    from paper_2407_19396_b200 import spec_of
    s = spec_of(env_id)
    assert (s.height, s.width, s.max_steps, s.n_actions, s.family, s.obs_bytes, s.view) == (h, w, T, na, fam, 147, 7)
    o = oracle_spec(env_id)  # the two independent parsers agree
    assert (o.height, o.width, o.max_steps, o.n_actions, o.export_bytes) == (h, w, T, na, s.export_bytes)
    assert o.family == fam


def test_unknown_ids_and_row_f2_sizes():
    from paper_2407_19396_b200 import NavixError, spec_of
    with pytest.raises(NavixError) as e:
        spec_of("Navix-NoSuchEnv-v0")
    assert e.value.status == 1 and "unknown env id" in str(e.value)
    for env_id, hw, T, nob in (("Navix-DoorKey-16x16-v0", 16, 2560, 0), ("Navix-Empty-16x16-v0", 16, 1024, 0),
                               ("Navix-Dynamic-Obstacles-16x16", 16, 1024, 8), ("KeyCorridorS4R3", 10, 480, 0),
                               ("KeyCorridorS5R3", 13, 750, 0), ("Navix-KeyCorridorS6R3-v0", 16, 1080, 0)):
        s = spec_of(env_id)  # row f2: grids up to 16x16 have kernels
        assert (s.height, s.width, s.max_steps, s.n_obstacles) == (hw, hw, T, nob), env_id


def test_argument_validation_before_any_cuda_call():
    from paper_2407_19396_b200 import load_library, state_bytes
    lib = load_library()
    h = ctypes.c_void_p()
    assert lib.navix_create_shard(b"DoorKey-8x8-v0", 10, 5, 10, 0, 0, None, 0, ctypes.byref(h)) == 2
    assert b"outside" in lib.navix_last_error()
    assert lib.navix_create_shard(b"DoorKey-8x8-v0", 10, 0, 0, 0, 0, None, 0, ctypes.byref(h)) == 2
    assert lib.navix_create_shard(b"DoorKey-8x8-v0", 10, 0, 10, 0, 0, None, 7, ctypes.byref(h)) == 2
    assert lib.navix_step(None, None, None, None, None, None, None) == 2
    assert lib.navix_reset(None, None, None) == 2
    assert state_bytes("DoorKey-8x8-v0", 0) == 0
    assert state_bytes("DoorKey-8x8-v0", 1 << 20) >= (1 << 20) * (64 + 8 + 4)
    assert state_bytes("Foo", 10) == 0
    assert lib.navix_create_shard(b"DoorKey-8x8-v0", 1 << 33, 0, 10, 0, 0, None, 0, ctypes.byref(h)) == 2
    assert b"2^32" in lib.navix_last_error()
    assert lib.navix_create_shard(None, 10, 0, 10, 0, 0, None, 0, ctypes.byref(h)) == 1
    assert lib.navix_set_observation(None, 1) == 2
    assert lib.navix_set_event_functions(None, 7, 7) == 2
    assert lib.navix_set_reward_costs(None, 0.0, 0.0) == 2
    assert lib.navix_rollout_random(None, 1, 0, 4, None, None, None, None, None) == 2
    assert lib.navix_reset_seed(None, 1, None, None) == 2


def test_shard_ranges_partition():
    from paper_2407_19396_b200 import shard_range
    for n in (1, 7, 1000, 1 << 23):
        for G in (1, 2, 3, 4, 8):
            if G > n:
                continue
            rs = [shard_range(n, r, G) for r in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def test_every_id_the_library_accepts_the_oracle_parses_identically():
    # the two independent id parsers: whatever libnavix accepts (one id per
    # kernel instantiation, many spellings), the oracle parses to the same spec
    from oracle import spec_of as oracle_spec
    from paper_2407_19396_b200 import NavixError, spec_of
    fams = ["Empty-{s}x{s}", "Empty-Random-{s}x{s}", "DoorKey-{s}x{s}", "DoorKey-Random-{s}x{s}",
            "Dynamic-Obstacles-{s}x{s}", "Dynamic-Obstacles-Random-{s}x{s}", "LavaGapS{s}", "GoToDoor-{s}x{s}",
            "KeyCorridorS{s}R1", "KeyCorridorS{s}R2", "KeyCorridorS{s}R3", "SimpleCrossingS{s}N1",
            "SimpleCrossingS{s}N2", "SimpleCrossingS{s}N3", "SimpleCrossingS{s}N5", "Crossings-S{s}N1",
            "Crossings-S{s}N2", "Crossings-S{s}N3", "Crossings-S{s}N5", "LavaCrossingS{s}N1", "LavaCrossingS{s}N2",
            "LavaCrossingS{s}N3", "LavaCrossingS{s}N5", "LavaGap-S{s}"]
    extra = ["FourRooms", "DistShift1", "DistShift2"]
    accepted = 0
    for pre in ("", "Navix-", "MiniGrid-"):
        for suf in ("", "-v0"):
            ids = [pre + f.format(s=s) + suf for f in fams for s in range(2, 19)] + [pre + e + suf for e in extra]
            for env_id in ids:
                try:
                    s = spec_of(env_id)
                except NavixError:
                    continue
                accepted += 1
                o = oracle_spec(env_id)
                assert (o.height, o.width, o.max_steps, o.n_actions, o.family, o.export_bytes, o.n_obstacles) == \
                    (s.height, s.width, s.max_steps, s.n_actions, s.family, s.export_bytes, s.n_obstacles), env_id
    # 54 kernel-backed ids (every Table 8 / 9 id, plus DoorKey / Dynamic-Obstacles
    # -Random at every size, the three Crossing and two LavaGap spellings) x 6 spellings
    assert accepted == 6 * 54


# Every env id printed in Table 8 and Table 9, verbatim
# (the duplicated Dynamic-Obstacles rows and the stray "N" of P:952 dropped, R#26).
TABLE8 = ["Navix-Empty-5x5-v0", "Navix-Empty-6x6-v0", "Navix-Empty-8x8-v0", "Navix-Empty-16x16-v0",
          "Navix-Empty-Random-5x5", "Navix-Empty-Random-6x6", "Navix-DoorKey-5x5-v0", "Navix-DoorKey-6x6-v0",
          "Navix-DoorKey-8x8-v0", "Navix-DoorKey-16x16-v0", "Navix-FourRooms-v0", "Navix-KeyCorridorS3R1-v0",
          "Navix-KeyCorridorS3R2-v0", "Navix-KeyCorridorS3R3-v0", "Navix-KeyCorridorS4R3-v0",
          "Navix-KeyCorridorS5R3-v0", "Navix-KeyCorridorS6R3-v0", "Navix-LavaGapS5-v0", "Navix-LavaGapS6-v0",
          "Navix-LavaGapS7-v0", "Navix-SimpleCrossingS9N1-v0", "Navix-SimpleCrossingS9N2-v0",
          "Navix-SimpleCrossingS9N3-v0", "Navix-SimpleCrossingS11N5-v0", "Navix-Dynamic-Obstacles-5x5",
          "Navix-Dynamic-Obstacles-6x6", "Navix-Dynamic-Obstacles-8x8", "Navix-Dynamic-Obstacles-16x16",
          "Navix-DistShift1-v0", "Navix-DistShift2-v0"]
TABLE9 = ["Navix-Empty-5x5-v0", "Navix-Empty-6x6-v0", "Navix-Empty-8x8-v0", "Navix-Empty-16x16-v0",
          "Navix-Empty-Random-5x5", "Navix-Empty-Random-6x6", "Navix-Empty-Random-8x8", "Navix-Empty-Random-16x16",
          "Navix-DoorKey-5x5-v0", "Navix-DoorKey-6x6-v0", "Navix-DoorKey-8x8-v0", "Navix-DoorKey-16x16-v0",
          "Navix-DoorKey-Random-5x5", "Navix-DoorKey-Random-6x6", "Navix-DoorKey-Random-8x8",
          "Navix-DoorKey-Random-16x16", "Navix-FourRooms-v0", "Navix-KeyCorridorS3R1-v0", "Navix-KeyCorridorS3R2-v0",
          "Navix-KeyCorridorS3R3-v0", "Navix-KeyCorridorS4R3-v0", "Navix-KeyCorridorS5R3-v0",
          "Navix-KeyCorridorS6R3-v0", "Navix-LavaGap-S5-v0", "Navix-LavaGap-S6-v0", "Navix-LavaGap-S7-v0",
          "Navix-Crossings-S9N1-v0", "Navix-Crossings-S9N2-v0", "Navix-Crossings-S9N3-v0", "Navix-Crossings-S11N5-v0",
          "Navix-Dynamic-Obstacles-5x5", "Navix-Dynamic-Obstacles-6x6", "Navix-Dynamic-Obstacles-8x8",
          "Navix-Dynamic-Obstacles-16x16", "Navix-DistShift1-v0", "Navix-DistShift2-v0", "Navix-GoToDoor-5x5-v0",
          "Navix-GoToDoor-6x6-v0", "Navix-GoToDoor-8x8-v0"]


@pytest.mark.parametrize("env_id", sorted(set(TABLE8 + TABLE9)))
def test_every_table8_table9_id_has_a_kernel(env_id):
    # navix_spec_of returns NAVIX_OK only for ids with a kernel instantiation
    # (NAVIX_E_UNSUPPORTED otherwise); the oracle parses the same spec
    from oracle import spec_of as oracle_spec
    from paper_2407_19396_b200 import load_library
    from paper_2407_19396_b200.navix import _Spec
    s = _Spec()
    assert load_library().navix_spec_of(env_id.encode(), ctypes.byref(s)) == 0, env_id
    o = oracle_spec(env_id)
    assert (o.height, o.width, o.max_steps) == (s.height, s.width, s.max_steps)
