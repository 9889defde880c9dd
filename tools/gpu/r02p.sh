# measurement box, branch-free form: host enqueue cost and A/B
set -x
for lib in libvxm_nobox.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python tools/host_enqueue_probe.py 64
done > gpurun_out/r02p_host.txt 2>&1
for rep in 1 2; do
for lib in libvxm_nobox.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'])"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg2:64,cfg1:64" timeout 300 python tools/quick_time.py 2>&1 | grep -A1 graph
done
done > gpurun_out/r02p_ab.txt 2>&1
cat gpurun_out/r02p_host.txt gpurun_out/r02p_ab.txt
