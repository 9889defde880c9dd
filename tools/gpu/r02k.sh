# re-entry check: full -m gpu suite, smoke, bench + reference arm on the committed code
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02k_bench_reference.json 2> gpurun_out/r02k_bench_reference.err
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02k_all.txt
tail -3 gpurun_out/r02k_smoke.txt gpurun_out/r02k_bench.err
cat gpurun_out/r02k_all.txt
