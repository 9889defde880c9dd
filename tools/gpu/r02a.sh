set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 900 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_trajectory.py tests/test_gpu_sequence.py tests/test_gpu_bench_multi.py -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r02a_newtests.txt
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
tail -3 gpurun_out/r02a_bench.err
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r02a_alltests.txt
cat gpurun_out/r02a_newtests.txt gpurun_out/r02a_alltests.txt
