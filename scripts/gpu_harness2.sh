python - <<'PY'
import json, subprocess, time, gzip, shutil, tempfile, os
from pathlib import Path
tmp = Path(tempfile.mkdtemp()); src = tmp / "s.jsonl"
with gzip.open("tests/golden/harvest/store10k.jsonl.gz","rb") as f, open(src,"wb") as g: shutil.copyfileobj(f,g)
def run(b, rounds, store, env=None):
    sc = json.loads(Path("tests/golden/scenarios/steady3.json").read_text()); sc["rounds"]=rounds
    if store:
        st = tmp / "x.jsonl"; shutil.copyfile(src, st); sc["experience_path"]=str(st)
    p = tmp/"sc.json"; p.write_text(json.dumps(sc))
    t0=time.perf_counter(); r=subprocess.run(["oracle/_ref/"+b, str(p), str(tmp/"l.csv")], capture_output=True, text=True, env=env); dt=time.perf_counter()-t0
    return round(dt,3)
for b in ("harness_b200","harness_ref"):
    print(b, "1 round no store", run(b, 1, False), "| 1 round 10k store", run(b, 1, True), "| 20 rounds 10k", run(b, 20, True), "| 60 rounds 10k", run(b, 60, True))
env = dict(os.environ, CUDA_MODULE_LOADING="LAZY")
print("b200 lazy", run("harness_b200", 1, False, env), run("harness_b200", 20, True, env))
env = dict(os.environ, SAIR_TRACE_DECISION="1")
PY
