#!/bin/bash
# K1 leaf-block variant scan (diagnostics): tools/scan_fused.py against every
# variant library built by paper_1701_03512_b200.build.build_variant, and the
# main library over the unit-size override.
O=${1:-gpurun_out/scan_gray.log}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O
for so in paper_1701_03512_b200/_lib/variants/*.so; do
  BINPATHS_LIB=$so timeout 300 python tools/scan_fused.py >> $O 2>&1
done
for u in 12 13 14 15; do
  BINPATHS_UNIT_LOG2=$u timeout 300 python tools/scan_fused.py >> $O 2>&1
done
