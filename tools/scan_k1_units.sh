#!/bin/bash
# tools/scan_k1.py over unit sizes (BINPATHS_UNIT_LOG2) for the main library and the variants
O=${1:-gpurun_out/scan_k1_units.log}
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader > $O
for u in 13 14 15; do
  echo "unit_log2=$u" >> $O
  BINPATHS_UNIT_LOG2=$u timeout 200 python tools/scan_k1.py >> $O 2>&1
  for so in paper_1701_03512_b200/_lib/variants/*.so; do BINPATHS_UNIT_LOG2=$u BINPATHS_LIB=$so timeout 200 python tools/scan_k1.py >> $O 2>&1; done
done
