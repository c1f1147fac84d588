"""configs[0] on the reference's bundled traces: the reference's unmodified
decision loop (harness.cpp) over a 10k-record experience store harvested from
the bundled scenarios (tests/golden/harvest), linked with the reference's own
experience/pareto/reward.cpp (oracle/_ref/harness_ref) and with the drop-in
(oracle/_ref/harness_b200).  Each run loads the store, replays R rounds of a
scenario (select + veto + reward + frontier update + store per decision) and
persists the store; wall time per decision, and the episode logs must be
byte-identical.  Prints one JSON line."""
import gzip
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
STORE = ROOT / "tests" / "golden" / "harvest" / "store10k.jsonl.gz"
SCEN = sorted((ROOT / "tests" / "golden" / "scenarios").glob("*.json"))


def run(binary, scenario, store_src, rounds, tmp, tag, env=None):
    store = tmp / f"{tag}.jsonl"
    shutil.copyfile(store_src, store)
    sc = json.loads(scenario.read_text())
    sc["rounds"] = rounds
    sc["experience_path"] = str(store)
    p = tmp / f"{tag}.json"
    p.write_text(json.dumps(sc))
    log = tmp / f"{tag}.csv"
    t0 = time.perf_counter()
    r = subprocess.run([str(binary), str(p), str(log)], capture_output=True, text=True,
                       timeout=3600, env=env)
    dt = time.perf_counter() - t0
    assert r.returncode == 0, r.stderr
    return dt, log.read_bytes(), store.read_bytes()


def main():
    rounds = int(os.environ.get("ROUNDS", 20))
    tmp = Path(tempfile.mkdtemp())
    src = tmp / "store.jsonl"
    with gzip.open(STORE, "rb") as f, open(src, "wb") as g:
        shutil.copyfileobj(f, g)
    n = sum(1 for _ in open(src))
    res = {"workload": f"configs[0] on the bundled traces: {n}-record store, {rounds} rounds x "
                       f"{len(SCEN)} scenarios", "records": n, "runs": []}
    for sc in SCEN:
        tb, lb, sb = run(ROOT / "oracle" / "_ref" / "harness_b200", sc, src, rounds, tmp, "b200")
        tr, lr, sr = run(ROOT / "oracle" / "_ref" / "harness_ref", sc, src, rounds, tmp, "ref")
        res["runs"].append({"scenario": sc.stem, "b200_s": round(tb, 3), "ref_s": round(tr, 3),
                            "identical_log": lb == lr, "identical_store": sb == sr})
    tb = sum(r["b200_s"] for r in res["runs"])
    tr = sum(r["ref_s"] for r in res["runs"])
    dec = rounds * len(SCEN)
    res.update({"b200_ms_per_decision": round(tb / dec * 1e3, 3),
                "ref_ms_per_decision": round(tr / dec * 1e3, 3),
                "speedup": round(tr / tb, 2),
                "note": "wall time of whole runs (process start, store load/persist included)"})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
