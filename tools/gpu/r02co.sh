set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02co_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02co_pytest.txt 2>&1
bash tools/profile_round.sh r02co > gpurun_out/r02co_prof.log 2>&1
timeout 900 python bench.py > gpurun_out/r02co_bench.json 2> gpurun_out/r02co_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02co_bench_reference.json 2> gpurun_out/r02co_bench_reference.err
timeout 300 python tools/host_enqueue_probe.py 64 > gpurun_out/r02co_host.txt 2>&1
tail -n 1 gpurun_out/r02co_smoke.txt
tail -n 3 gpurun_out/r02co_pytest.txt
