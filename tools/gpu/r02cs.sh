# K2 z-OR as a sliding window over registers (libvxm) vs HEAD
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_bench_parity.py tests/test_gpu_keys.py -x -q -m gpu 2>&1 | tail -2 > gpurun_out/r02cs_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:64,cfg2:1,cfg2:8" timeout 600 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02cs_ab.txt 2>&1
for lib in libvxm_head.so libvxm.so libvxm_head.so libvxm.so; do VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib bench value', d['value'], 'stage', d['stage_ms_per_step'])"; done >> gpurun_out/r02cs_ab.txt 2>&1
cat gpurun_out/r02cs_tests.txt; grep -v "^cfg" gpurun_out/r02cs_ab.txt
