# K1 dense path: quad pixels transformed 2 (libvxm) or 4 (pb4) at a time, exact-floor pixels deferred (A/B vs HEAD)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02bt_tests.txt
VXM_LIB_NAME=libvxm_pb4.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "k1 or depth or special" 2>&1 | tail -3 >> gpurun_out/r02bt_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm.so libvxm_pb4.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:64,cfg1:1,cfg3:16,cfg2:64" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02bt_ab.txt 2>&1
cat gpurun_out/r02bt_tests.txt; grep -v stages gpurun_out/r02bt_ab.txt
