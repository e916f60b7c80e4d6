for v in nu8_4 nu8_8; do
  echo "== $v"
  VCA_LIB=paper_2304_12384_b200/variants/libvca_$v.so python tools/family_sweep.py 2>&1 | grep -E '"block": (8|16), "lowpass": (true|false), "path": "fused' | grep -E '"block": 8|"lowpass": true'
  VCA_LIB=paper_2304_12384_b200/variants/libvca_$v.so timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "lp16 or full8" 2>&1 | tail -n 1
done
