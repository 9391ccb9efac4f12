#!/bin/bash
# Round profiling pass (run under gpurun, ONE GPU).  Every command first runs
# without ncu and must exit 0; then the launch list of one bench run and one
# ncu --set full capture per dominant kernel.  Output: gpurun_out/prof/.
set -u
O=${1:-gpurun_out/prof}
mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
run() { echo "== $*" >> $O/runs.log; timeout 600 "$@" >> $O/runs.log 2>&1; echo "rc=$?" >> $O/runs.log; }
run python tools/profile_exact.py config2 3
run python tools/profile_exact.py config3 2
run python tools/scan_mc_batch.py mc
run python tools/scan_mc_batch.py batch
run python bench.py --steps 3 --warmup 3 --no-config3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config2.csv \
  python bench.py --steps 3 --warmup 3 --no-config3 > $O/ncu_launches.log 2>&1
timeout 600 $NCU -k regex:k_exact_fast -s 1 -c 1 -o $O/config2_full python tools/profile_exact.py config2 3 > $O/ncu_c2.log 2>&1
timeout 600 $NCU -k regex:k_exact_fast -s 1 -c 1 -o $O/config3_full python tools/profile_exact.py config3 2 > $O/ncu_c3.log 2>&1
timeout 600 $NCU -k regex:k_mc_strata -s 2 -c 1 -o $O/mc_full python tools/scan_mc_batch.py mc > $O/ncu_mc.log 2>&1
timeout 600 $NCU -k regex:k_exact_batch -s 1 -c 1 -o $O/batch_full python tools/scan_mc_batch.py batch > $O/ncu_batch.log 2>&1
echo done >> $O/runs.log
