"""Harvest configs[0]'s experience store from the reference's bundled
scenarios (proj/scenarios/*.json): the reference's own decision loop
(oracle/_ref/harness_ref: harness.cpp with the reference's
experience/pareto/reward.cpp, compiled in place) replays each scenario with a
persistent experience_path (harness.cpp:152-153 loads it, :329 persists it),
seed after seed, round-robin over the three scenarios, until the buffer holds
TARGET records.  Run here, where /root/reference exists; the JSONL it writes
(store10k.jsonl.gz) is the fixture -- the reference's own persistence format
(experience.cpp:207-271).

    python tests/golden/harvest/make_store.py [TARGET]
"""
import gzip
import json
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[3]
REF = ROOT / "oracle" / "_ref" / "harness_ref"
SCEN = sorted(Path("/root/reference/proj/scenarios").glob("*.json"))
OUT = Path(__file__).resolve().parent / "store10k.jsonl.gz"


def main(target: int = 10000, rounds: int = 400):
    tmp = Path(tempfile.mkdtemp())
    store = tmp / "store.jsonl"
    n, seed, runs = 0, 1000, []
    while n < target:
        for sp in SCEN:
            sc = json.loads(sp.read_text())
            sc["seed"] = seed
            sc["rounds"] = rounds
            sc["experience_path"] = str(store)
            p = tmp / f"{sp.stem}.json"
            p.write_text(json.dumps(sc))
            r = subprocess.run([str(REF), str(p), str(tmp / "log.csv")], capture_output=True,
                               text=True, timeout=3600)
            assert r.returncode == 0, r.stderr
            n = sum(1 for _ in open(store)) if store.exists() else 0
            runs.append((sp.name, seed, n))
            print(f"{sp.name} seed {seed}: {n} records", flush=True)
            if n >= target:
                break
        seed += 1
    with open(store, "rb") as f, gzip.open(OUT, "wb", compresslevel=9) as g:
        shutil.copyfileobj(f, g)
    (OUT.parent / "runs.json").write_text(json.dumps({"rounds": rounds, "runs": runs}, indent=0))
    print(f"wrote {OUT} ({n} records)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10000)
