# K3 fast chunks (per-axis bound, fma step, clone lanes, snap counters): parity, then A/B vs the committed K3
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keys.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r02l_parity.txt
cat gpurun_out/r02l_parity.txt
for rep in 1 2; do
for lib in libvxm_old.so libvxm.so libvxm_m20.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'], 'parity', d.get('parity_ok'))"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg1:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep graph
done
done > gpurun_out/r02l_ab.txt 2>&1
cat gpurun_out/r02l_ab.txt
