set -x
bash tools/profile_round.sh r02aj > gpurun_out/r02aj_prof.log 2>&1
timeout 900 python bench.py > gpurun_out/r02aj_bench.json 2> gpurun_out/r02aj_bench.err
timeout 300 python bench.py --impl reference > gpurun_out/r02aj_bench_reference.json 2> gpurun_out/r02aj_bench_reference.err
