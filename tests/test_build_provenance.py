"""Build provenance: the libnavix.so under test was compiled from THIS tree.

build.py hashes every CUDA source, header and compiler flag into a build id
compiled into the library (navix_build_id, include/navix.h); a prebuilt or
stale .so that does not match the checked-out sources fails here (and
build() rebuilds it, since staleness is decided by the id, not by mtimes)."""
import os
import shutil

import pytest


def _check_tree_matches_library():
    from paper_2407_19396_b200 import build_id
    from paper_2407_19396_b200.build import embedded_build_id, source_hash
    want = source_hash()
    assert embedded_build_id() == want, "libnavix.so on disk was built from other sources: run build()"
    assert build_id() == want, "the loaded libnavix.so was built from other sources"


def test_library_build_id_matches_tree():
    _check_tree_matches_library()


@pytest.mark.gpu
def test_library_build_id_matches_tree_on_gpu_box():
    _check_tree_matches_library()


def test_any_source_change_makes_the_library_stale(tmp_path, monkeypatch):
    from paper_2407_19396_b200 import build as b
    src = tmp_path / "pkg" / "csrc"  # HEADERS name ../../include/navix.h relative to csrc
    shutil.copytree(b.CSRC, src)
    shutil.copytree(os.path.join(b.CSRC, "..", "..", "include"), tmp_path / "include")
    monkeypatch.setattr(b, "CSRC", str(src))
    h0 = b.source_hash()
    assert h0 == b.embedded_build_id()  # same bytes, another directory: same id
    for name in b.SOURCES[:2] + ["step_kernel.cuh"]:
        p = src / name
        orig = p.read_bytes()
        p.write_bytes(orig + b"\n// touched\n")
        assert b.source_hash() != h0, name
        assert b._stale()
        p.write_bytes(orig)
    assert b.source_hash() == h0 and not b._stale()
    monkeypatch.setattr(b, "FLAGS", b.FLAGS + ["-DNAVIX_EXPERIMENT"])
    assert b.source_hash() != h0  # flags are part of the id
