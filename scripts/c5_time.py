"""configs[4]'s per-GPU decision step (bench.bench_decision_step) on a fresh 16M store."""
import os, sys, json
sys.path.insert(0, ".")
import bench
import paper_2601_22397_b200 as sair
buf = sair.ExperienceBuffer(0.0)
buf.store_synthetic(bench.SEED, bench.N_RECORDS, bench.DIM)
print(os.environ.get("TAG", ""), json.dumps(bench.bench_decision_step(buf, 0)), flush=True)
st = buf.last_stats()
print({k: st[k] for k in ("retried", "certified", "tensor_core", "qb", "candidates")}, flush=True)
