#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the smoke solve (c1-shaped, 200 docs)
# plus a small unfused + tol solve; logs in gpurun_out/sanitizer_<tool>.log
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import __graft_entry__ as g
g.smoke()
import paper_2107_06433_b200 as swmd
from paper_2107_06433_b200 import synth
inst = synth.zipf_instance("c1", n_docs=120)
c = inst.corpus()
a = swmd.unfused_sparse_wmd(inst.query, c, inst.embeddings, swmd.SolverConfig())
b = swmd.sinkhorn_wmd(inst.query, c, inst.embeddings, swmd.SolverConfig(lam=1.0, max_iter=40, tol=1e-9))
print("sanitizer case ok", a.shape, b.iterations_run)
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python /tmp/san_case.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "sanitizer_${tool}_rc=$?"; grep -E "ERROR SUMMARY|sanitizer case ok" gpurun_out/sanitizer_$tool.log | tail -2
done
