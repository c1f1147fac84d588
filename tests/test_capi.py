"""CPU-side checks of the drop-in boundary (no compute without a GPU)."""
import ctypes as C
import subprocess

import pytest

from paper_2601_22397_b200 import _lib


def test_header_declares_the_boundary():
    syms = _lib.header_symbols()
    for s in ("sair_store_create", "sair_store_append", "sair_store_select",
              "sair_store_effective_sigma", "sair_store_surprisal", "sair_store_nearest",
              "sair_frontier_create", "sair_frontier_update", "sair_frontier_insert_batch",
              "sair_frontier_score_batch", "sair_frontier_contribution",
              "sair_dominance_counts", "sair_compute_reward", "sair_compute_reward_batch",
              "sair_action_magnitude", "sair_last_error"):
        assert s in syms
    # the ctypes binding covers exactly the header
    assert sorted(_lib.SIGNATURES) == syms


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    for s in _lib.header_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(_lib.header_symbols()) <= exported
    # nothing but the C-ABI leaks out of the shared object
    assert all(e.startswith("sair_") for e in exported), sorted(e for e in exported
                                                                 if not e.startswith("sair_"))


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.lib()
    h = C.c_void_p()
    rc = L.sair_store_create(0.0, 0, 0, C.byref(h))
    assert rc == _lib.SAIR_ECUDA
    assert b"no CUDA device" in L.sair_last_error()
    from paper_2601_22397_b200 import ExperienceBuffer, SairError
    with pytest.raises(SairError):
        ExperienceBuffer(0.0)


def test_status_codes_for_bad_arguments():
    L = _lib.lib()
    assert L.sair_store_create(0.0, 0, 0, None) == _lib.SAIR_EINVAL
    assert L.sair_store_size(None, None) == _lib.SAIR_EINVAL
    assert L.sair_store_destroy(None) == _lib.SAIR_OK


def test_similarity_is_the_references(ref):
    """sair_similarity (host arithmetic, like standardize) is bit-identical to
    the reference's similarity() (experience.cpp:30-40), including its errors."""
    import numpy as np
    L = _lib.lib()
    rng = np.random.default_rng(5)
    dp = C.POINTER(C.c_double)
    for d in (1, 7, 37, 64, 300):
        for _ in range(20):
            a, b = rng.normal(size=d) * 50, rng.normal(size=d) * 50
            sig = float(rng.uniform(0.5, 200))
            got, want = C.c_double(), C.c_double()
            assert L.sair_similarity(a.ctypes.data_as(dp), d, b.ctypes.data_as(dp), d, sig,
                                     C.byref(got)) == _lib.SAIR_OK
            assert ref.lib.ref_similarity(a.ctypes.data_as(dp), b.ctypes.data_as(dp), d, d, sig,
                                          C.byref(want)) == 0
            assert got.value == want.value
    a = np.zeros(3)
    out = C.c_double()
    assert L.sair_similarity(a.ctypes.data_as(dp), 3, a.ctypes.data_as(dp), 2, 1.0,
                             C.byref(out)) == _lib.SAIR_EINVAL
    assert L.sair_similarity(a.ctypes.data_as(dp), 3, a.ctypes.data_as(dp), 3, 0.0,
                             C.byref(out)) == _lib.SAIR_EINVAL


def test_multigpu_entry_points_fail_loudly_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = _lib.lib()
    devs = (C.c_int * 2)(0, 1)
    h = C.c_void_p()
    assert L.sair_comm_create(devs, 2, C.byref(h)) == _lib.SAIR_ECUDA
    assert L.sair_comm_destroy(None) == _lib.SAIR_OK
    assert L.sair_sharded_create(None, 0.0, 10, C.byref(h)) == _lib.SAIR_EINVAL
