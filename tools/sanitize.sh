#!/bin/bash
# compute-sanitizer over small pipeline runs (memcheck: out-of-bounds /
# misaligned accesses; racecheck: shared-memory hazards in the staged kernels;
# synccheck). Output -> gpurun_out/sanitizer_*.txt
mkdir -p gpurun_out
PY="python tools/sanitize_case.py"
compute-sanitizer --tool memcheck --leak-check full $PY > gpurun_out/sanitizer_memcheck.txt 2>&1
compute-sanitizer --tool racecheck --racecheck-report all $PY > gpurun_out/sanitizer_racecheck.txt 2>&1
compute-sanitizer --tool synccheck $PY > gpurun_out/sanitizer_synccheck.txt 2>&1
compute-sanitizer --tool initcheck $PY > gpurun_out/sanitizer_initcheck.txt 2>&1
tail -n 3 gpurun_out/sanitizer_*.txt
