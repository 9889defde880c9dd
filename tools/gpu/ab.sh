# Generic GPU round trip: parity tests, then A/B of library builds.
#   bash tools/gpu/ab.sh TAG "pytest args or -" REPS lib1.so lib2.so ...
TAG=$1; TESTS=$2; REPS=$3; shift 3
if [ "$TESTS" != "-" ]; then
  timeout 1800 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -4 > gpurun_out/${TAG}_tests.txt
fi
for rep in $(seq $REPS); do
for lib in "$@"; do
  echo "== $lib"
  VXM_LIB_NAME=$lib timeout 300 python bench.py --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench value', d['value'], 'stage', d['stage_ms_per_step'])"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:1,cfg1:64,cfg3:16" timeout 300 python tools/quick_time.py 2>&1 | grep graph
done
done > gpurun_out/${TAG}_ab.txt 2>&1
cat gpurun_out/${TAG}_tests.txt gpurun_out/${TAG}_ab.txt 2>/dev/null
