#!/bin/bash
# One GPU iteration: the GPU tests (first failures only), a bench line, and
# (with a second argument "ncu") a full capture of the headline kernel.
O=gpurun_out/${1:-iter}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --maxfail=1 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
if [ "$2" = "ncu" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 \
    -o $O/config2_full python tools/profile_exact.py config2 3 > $O/ncu_c2.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 \
    -o $O/config3_full python tools/profile_exact.py config3 2 > $O/ncu_c3.log 2>&1
fi
echo done
