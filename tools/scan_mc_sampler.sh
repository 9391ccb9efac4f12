#!/bin/bash
# K4 (config 4) under draws-per-thread x resident-CTA variants of the bit-sliced sampler -> gpurun_out/$1/scan.log
O=gpurun_out/${1:-mc_scan}; mkdir -p $O
echo "== main" >> $O/scan.log
python tools/scan_mc_batch.py 2>&1 | head -2 >> $O/scan.log
for so in paper_1701_03512_b200/_lib/variants/mc_ns*.so; do
  echo "== $so" >> $O/scan.log
  BINPATHS_LIB=$so python tools/scan_mc_batch.py 2>&1 | head -2 >> $O/scan.log
done
