# A/B: interleaved fast-chunk loads (default), parallel compares, branch counts, register cap
for rep in 1 2; do
for lib in libvxm.so libvxm_il0.so libvxm_pc1.so libvxm_br2.so libvxm_br4.so libvxm_m24.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'])"
done
done > gpurun_out/r02n_ab.txt 2>&1
cat gpurun_out/r02n_ab.txt
