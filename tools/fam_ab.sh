#!/bin/bash
# A/B of the n = 8 / 16 families (1080p, 720p; tools/family_sweep.py) over the builds in
# paper_2304_12384_b200/variants/ (VCA_LIB selects the library).
for v in paper_2304_12384_b200/variants/*.so; do
  for rep in 1 2; do
    echo "== $(basename $v) round $rep"
    VCA_LIB=$v timeout 300 python tools/family_sweep.py 2>&1 | grep -E '"block": (8|16)' | grep -E '"W": (1920|1280)'
  done
done
