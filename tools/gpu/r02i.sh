for rep in 1 2; do
for lib in libvxm.so libvxm_pipe24.so libvxm_pipe20.so libvxm_pipe16.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'])"
done
done > gpurun_out/r02i_ab.txt 2>&1
VXM_LIB_NAME=libvxm_pipe16.so timeout 600 python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/r02i_ab.txt
cat gpurun_out/r02i_ab.txt
