# final validation at HEAD: gpu tests, smoke, bench, reference arm
mkdir -p gpurun_out
T=r02df
(timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.txt 2>&1; echo "exit $?" >> gpurun_out/${T}_gpu_tests.txt)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 400 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err
tail -3 gpurun_out/${T}_gpu_tests.txt; tail -1 gpurun_out/${T}_smoke.txt
