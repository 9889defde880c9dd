set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cl_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02cl_pytest.txt 2>&1
bash tools/profile_round.sh r02cl > gpurun_out/r02cl_prof.log 2>&1
timeout 900 python bench.py > gpurun_out/r02cl_bench.json 2> gpurun_out/r02cl_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02cl_bench_reference.json 2> gpurun_out/r02cl_bench_reference.err
timeout 300 python tools/host_enqueue_probe.py 64 > gpurun_out/r02cl_host.txt 2>&1
tail -n 1 gpurun_out/r02cl_smoke.txt
tail -n 3 gpurun_out/r02cl_pytest.txt
