VXM_LIB_NAME=libvxm_dmax1024.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_bench_parity.py -x -q -m gpu 2>&1 | tail -2
for rep in 1 2; do for lib in libvxm.so libvxm_dmax1024.so; do
  echo "== $lib"; VXM_LIB_NAME=$lib QT_CONFIGS="cfg3:16,cfg2:64" timeout 300 python tools/quick_time.py 2>&1 | grep -A1 graph
done; done
