# chain merge publishes its counters (no K5 on the range chain); K4 lone-frame rows per warp >= 4 (rpw4)
timeout 1200 python -m pytest tests/test_gpu_sequence.py tests/test_gpu_trajectory.py tests/test_gpu_keys.py tests/test_dropin_cpp.py tests/test_gpu_bench_parity.py -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r02br_tests.txt
VXM_LIB_NAME=libvxm_rpw4.so timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3 >> gpurun_out/r02br_tests.txt
for rep in 1 2; do for lib in libvxm_head.so libvxm.so libvxm_rpw4.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg1:1,cfg3:1,cfg1:1:64,cfg2:1:64,cfg2:64" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^$"
done; done > gpurun_out/r02br_ab.txt 2>&1
cat gpurun_out/r02br_tests.txt; grep -v stages gpurun_out/r02br_ab.txt
