# merge4 key decode with byte permutes (prmt) vs HEAD, bench value included
VXM_LIB_NAME=libvxm_prmt.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_bench_parity.py tests/test_gpu_keys.py tests/test_gpu_sequence.py tests/test_gpu_trajectory.py -x -q -m gpu 2>&1 | tail -2 > gpurun_out/r02cq_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm_prmt.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:64,cfg1:64,cfg3:16,cfg2:8" timeout 600 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02cq_ab.txt 2>&1
for lib in libvxm_head.so libvxm_prmt.so libvxm_head.so libvxm_prmt.so; do VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib bench value', d['value'], 'stage', d['stage_ms_per_step'])"; done >> gpurun_out/r02cq_ab.txt 2>&1
cat gpurun_out/r02cq_tests.txt; grep -v stages gpurun_out/r02cq_ab.txt
