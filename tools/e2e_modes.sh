#!/bin/bash
# e2e of value_exact (config 2) under the synchronous path's toggles -> gpurun_out/$1
O=gpurun_out/${1:-e2e_modes}; mkdir -p $O
for m in "1 0" "0 0" "1 1" "0 1" "1 0" "0 0"; do
  set -- $m
  echo "== BINPATHS_MAPPED_OUT=$1 BINPATHS_GRAPH_EVENTS=$2" >> $O/modes.log
  BINPATHS_MAPPED_OUT=$1 BINPATHS_GRAPH_EVENTS=$2 python tools/e2e_probe.py 2>&1 | head -3 >> $O/modes.log
done
BINPATHS_TRACE=1 python - >> $O/modes.log 2>&1 <<'PY'
import bench, paper_1701_03512_b200 as bp
wl, crr = bench.workloads()
req, kinds, _ = bench.make_req(wl["config2"], crr)
for i in range(6):
    r = bp.value_exact(req, kinds=kinds, devices=[0])
print(r.values)
PY
