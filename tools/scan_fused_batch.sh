for so in paper_1701_03512_b200/_lib/variants/*.so; do
  BINPATHS_LIB=$so timeout 120 python tools/scan_fused.py
  echo "$(basename $so) $(BINPATHS_LIB=$so timeout 120 python tools/scan_mc_batch.py batch)"
done
timeout 120 python tools/scan_fused.py; echo "main $(timeout 120 python tools/scan_mc_batch.py batch)"
