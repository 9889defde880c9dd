# A/B: K3 key REDs with an L2 evict-last policy
mkdir -p gpurun_out
AB=gpurun_out/r02de_k3_red_evict_last_ab.txt
for rep in 1 2 3; do
for lib in libvxm.so libvxm_redh.so; do
  echo "== $lib" >> $AB
  VXM_LIB_NAME=$lib QT_CONFIGS=cfg2:64,cfg1:64 timeout 200 python tools/quick_time.py 2>&1 | grep -A1 x64 >> $AB
  VXM_LIB_NAME=$lib timeout 200 python bench.py --no-extras --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib bench value', d['value'], d.get('stage_ms_per_step'))" >> $AB
done
done
