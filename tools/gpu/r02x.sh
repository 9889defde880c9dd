set -x
timeout 900 python bench.py > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02x_bench_reference.json 2> gpurun_out/r02x_bench_reference.err
tail -2 gpurun_out/r02x_bench.err
