for rep in 1 2; do
for lib in libvxm.so libvxm_prio.so libvxm_prio4.so libvxm_prio2.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'], 'e2e', d['e2e']['value'])"
done
done > gpurun_out/r02g_ab.txt 2>&1
for lib in libvxm.so libvxm_prio.so; do echo "== $lib"; VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep graph; done >> gpurun_out/r02g_ab.txt 2>&1
cat gpurun_out/r02g_ab.txt
