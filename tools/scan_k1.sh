#!/bin/bash
# tools/scan_k1.py over the main library and every variant library
O=${1:-gpurun_out/scan_k1.log}
nvidia-smi --query-gpu=name,clocks.max.sm --format=csv,noheader > $O
timeout 300 python tools/scan_k1.py >> $O 2>&1
for so in paper_1701_03512_b200/_lib/variants/*.so; do BINPATHS_LIB=$so timeout 300 python tools/scan_k1.py >> $O 2>&1; done
timeout 300 python tools/scan_k1.py >> $O 2>&1
