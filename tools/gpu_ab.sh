# A/B all variants on the configs in $AB_CONFIGS (default "3 4 2")
mkdir -p gpurun_out
for c in ${AB_CONFIGS:-3 4 2}; do
  echo "=== config $c" >> gpurun_out/ab.log
  rm -f gpurun_out/ab_ref_${c}_*.npy
  AB_CONFIG=$c python tools/ab_variants.py >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
