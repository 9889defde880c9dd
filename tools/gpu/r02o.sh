# measurement box in K4: full gpu suite, then A/B vs the previous build
set -x
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r02o_all.txt
cat gpurun_out/r02o_all.txt
for rep in 1 2; do
for lib in libvxm_nobox.so libvxm.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'])"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg1:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep graph
done
done > gpurun_out/r02o_ab.txt 2>&1
cat gpurun_out/r02o_ab.txt
