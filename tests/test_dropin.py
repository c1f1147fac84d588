"""The C++ drop-in (paper_2601_22397_b200/cpp: the reference's scalelab
classes on libsair's C ABI).

* tests/cpp/test_scalelab_b200 restates the reference's unit and acceptance
  expectations for the path against the drop-in (exit status = failures).
* oracle/_ref/harness_ref and harness_b200 are the reference's unmodified
  decision loop (harness.cpp, policy.cpp, simulator.cpp, ...) linked with the
  reference's experience/pareto/reward.cpp and with the drop-in respectively.
  Equal seeds must give byte-identical episode logs -- the reference's own
  determinism criterion (tests/test_harness.cpp:142-150) -- which requires
  every selection, veto, reward and frontier update to match exactly.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_BIN = ROOT / "oracle" / "_ref" / "harness_ref"
B200_BIN = ROOT / "oracle" / "_ref" / "harness_b200"
CPP_TEST = ROOT / "tests" / "cpp" / "test_scalelab_b200"
SCEN = sorted((ROOT / "tests" / "golden" / "scenarios").glob("*.json"))


def _need(p):
    if not p.exists():
        pytest.skip(f"{p.name} not built (built where /root/reference exists)")


def test_reference_harness_runs_on_cpu(tmp_path):
    _need(REF_BIN)
    out = tmp_path / "log.csv"
    r = subprocess.run([str(REF_BIN), str(SCEN[0]), str(out)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert out.read_text().startswith("round,")


@pytest.mark.gpu
def test_cpp_dropin_meets_reference_expectations():
    _need(CPP_TEST)
    r = subprocess.run([str(CPP_TEST)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("devices", ["", "0,0"], ids=["one-gpu", "sharded"])
@pytest.mark.parametrize("scenario", SCEN, ids=[s.stem for s in SCEN])
def test_reference_decision_loop_identical_with_dropin(tmp_path, scenario, devices):
    """devices "0,0": the drop-in's select() runs over a buffer sharded over
    two GPU slots (SAIR_DEVICES; one B200 per test box, so both on device 0 --
    on a multi-GPU node the same run takes distinct GPUs over NCCL)."""
    import os
    _need(REF_BIN)
    _need(B200_BIN)
    a, b = tmp_path / "ref.csv", tmp_path / "b200.csv"
    ra = subprocess.run([str(REF_BIN), str(scenario), str(a)], capture_output=True, text=True,
                        timeout=600)
    env = dict(os.environ)
    if devices:
        env["SAIR_DEVICES"] = devices
    rb = subprocess.run([str(B200_BIN), str(scenario), str(b)], capture_output=True, text=True,
                        timeout=600, env=env)
    assert ra.returncode == 0, ra.stderr
    assert rb.returncode == 0, rb.stderr
    assert ra.stdout == rb.stdout  # run summary: p99 and frontier hypervolume
    assert a.read_bytes() == b.read_bytes()


def test_cpp_expectations_hold_for_the_reference_itself():
    """The same runner linked with the reference's own implementation: the
    restated expectations are the reference's (CPU, no GPU needed)."""
    exe = ROOT / "oracle" / "_ref" / "test_scalelab_ref"
    _need(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
