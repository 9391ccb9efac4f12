#!/bin/bash
# GPU validation pass (one GPU): the GPU tests, a bench line, the loud
# failure of --gpus 2 on a 1-GPU box, the reference arm.  -> gpurun_out/$1/
O=gpurun_out/${1:-check}; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
python bench.py --gpus 2 --steps 2 > $O/bench_gpus2.out 2> $O/bench_gpus2.err; echo "rc=$?" >> $O/bench_gpus2.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
