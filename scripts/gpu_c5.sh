TAG=default timeout 600 python scripts/c5_time.py 2>&1 | tail -1
SAIR_WIDE_BF16=0 TAG=tf32 timeout 600 python scripts/c5_time.py 2>&1 | tail -1
SAIR_WIDE_AGGR=0 TAG=safe timeout 600 python scripts/c5_time.py 2>&1 | tail -1
SAIR_WIDE_BF16=0 SAIR_WIDE_AGGR=0 TAG=tf32safe timeout 600 python scripts/c5_time.py 2>&1 | tail -1
for sc in steady3 bursty3; do for r in 0 20; do
python - <<PY
import json, subprocess, time, gzip, shutil, tempfile
from pathlib import Path
tmp = Path(tempfile.mkdtemp()); src = tmp / "s.jsonl"
with gzip.open("tests/golden/harvest/store10k.jsonl.gz","rb") as f, open(src,"wb") as g: shutil.copyfileobj(f,g)
for b in ("harness_b200","harness_ref"):
    st = tmp / "x.jsonl"; shutil.copyfile(src, st)
    sc = json.loads(Path("tests/golden/scenarios/$sc.json").read_text()); sc["rounds"]=$r; sc["experience_path"]=str(st)
    p = tmp/"sc.json"; p.write_text(json.dumps(sc))
    t0=time.perf_counter(); r=subprocess.run(["oracle/_ref/"+b, str(p), str(tmp/"l.csv")], capture_output=True, text=True); dt=time.perf_counter()-t0
    print("$sc rounds=$r", b, round(dt,3), r.returncode, r.stderr[-200:])
PY
done; done
