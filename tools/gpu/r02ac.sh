set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ac_smoke.txt 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r02ac_all.txt
bash tools/profile_round.sh r02ac > gpurun_out/r02ac_prof.log 2>&1
timeout 900 python bench.py > gpurun_out/r02ac_bench.json 2> gpurun_out/r02ac_bench.err
cat gpurun_out/r02ac_all.txt; tail -2 gpurun_out/r02ac_smoke.txt
