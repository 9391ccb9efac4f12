#!/bin/bash
# Full ncu captures of the headline kernels (config 2 fused K1, config 3 K1,
# config 5 K3, config 4 K4) and the launch list of the default bench command.
O=gpurun_out/${1:-prof}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 \
  -o $O/config2_full python tools/profile_exact.py config2 3 > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 \
  -o $O/config3_full python tools/profile_exact.py config3 2 > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_exact_batch -s 1 -c 1 \
  -o $O/config5_full python tools/scan_mc_batch.py > $O/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_mc_strata -s 1 -c 1 \
  -o $O/config4_full python tools/scan_mc_batch.py > $O/ncu_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-config3 > $O/ncu_launch.log 2>&1
echo done
