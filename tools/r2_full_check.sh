#!/bin/bash
# Round-2 validation on one GPU: the checks (tools/r2_gpu_check.sh), then a
# launch list of the bench command and a full capture of the headline kernel.
bash tools/r2_gpu_check.sh ${1:-r2check}
O=gpurun_out/${1:-r2check}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-config3 > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 \
  -o $O/config2_full python tools/profile_exact.py config2 3 > $O/ncu_c2.log 2>&1
echo done
