#!/bin/bash
# I15 screen scan (diagnostics): main library fused / unfused, and the
# variant libraries (BP_I15=0, occupancy targets).
O=${1:-gpurun_out/scan_i15.log}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O
timeout 300 python tools/scan_fused.py >> $O 2>&1
BINPATHS_FUSE_ACFL=0 timeout 300 python tools/scan_fused.py 2>&1 | sed 's/^/unfused /' >> $O
for so in paper_1701_03512_b200/_lib/variants/*.so; do
  BINPATHS_LIB=$so timeout 300 python tools/scan_fused.py >> $O 2>&1
  BINPATHS_LIB=$so BINPATHS_FUSE_ACFL=0 timeout 300 python tools/scan_fused.py 2>&1 | sed 's/^/unfused /' >> $O
done
