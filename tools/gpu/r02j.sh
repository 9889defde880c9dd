set -x
timeout 900 python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02j_bench_reference.json 2> gpurun_out/r02j_bench_reference.err
timeout 400 python tools/fuzz_parity.py 300 202 > gpurun_out/r02j_fuzz.txt 2>&1
timeout 200 python tools/fuzz_stages.py 150 203 > gpurun_out/r02j_fuzz_stages.txt 2>&1
timeout 300 python tools/host_enqueue_probe.py 64 > gpurun_out/r02j_host.txt 2>&1
tail -2 gpurun_out/r02j_fuzz.txt gpurun_out/r02j_fuzz_stages.txt gpurun_out/r02j_bench.err
cat gpurun_out/r02j_host.txt gpurun_out/r02j_bench_reference.json
