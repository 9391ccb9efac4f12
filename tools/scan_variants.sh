#!/bin/bash
# Run the exact-engine scan against every built variant .so (diagnostics).
for so in paper_1701_03512_b200/_lib/variants/*.so; do
  echo "== $so"
  BINPATHS_LIB=$so python tools/scan_exact.py 2>&1 | sed -n "1,4p;9p" | awk '{print $1, $3, $5, $6}'
done
