#!/bin/bash
# tools/scan_fused.py against every built variant .so (diagnostics)
for so in paper_1701_03512_b200/_lib/variants/*.so; do
  BINPATHS_LIB=$so timeout 120 python tools/scan_fused.py
done
