cd $GRAFT_REPO_ROOT
SAIR_DOM_STATS=1 timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import paper_2601_22397_b200 as sair
from paper_2601_22397_b200 import synth
for K, dist in [(3,'uniform'),(3,'uniform'),(4,'uniform'),(4,'corr'),(3,'grid')]:
    t = synth.tuples(2028+K, 4194304, K, dist)
    t0=time.perf_counter(); sair.dominance_counts(t); print(K, dist, time.perf_counter()-t0, flush=True)
" 2>&1
