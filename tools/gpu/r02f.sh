for lib in libvxm_old.so libvxm.so libvxm_old.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:64,cfg1:64" timeout 300 python tools/quick_time.py 2>&1 | grep -v "^\s*$"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'], 'e2e', d['e2e']['value'])"
done > gpurun_out/r02f_ab.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02f_all.txt
cat gpurun_out/r02f_ab.txt gpurun_out/r02f_all.txt
