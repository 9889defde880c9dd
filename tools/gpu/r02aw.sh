set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aw_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02aw_bench.json 2> gpurun_out/r02aw_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02aw_bench_reference.json 2> gpurun_out/r02aw_bench_reference.err
tail -1 gpurun_out/r02aw_smoke.txt
