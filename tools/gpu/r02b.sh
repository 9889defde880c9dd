# key-format change: parity first, then timing
set -x
timeout 600 python -m pytest tests/test_gpu_keys.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02b_keys.txt
timeout 600 python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_sequence.py tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02b_parity2.txt
QT_CONFIGS="cfg2:64,cfg1:64,cfg3:16,cfg2:1" timeout 300 python tools/quick_time.py > gpurun_out/r02b_qt.txt 2>&1
QT_FLAGS=64 QT_CONFIGS="cfg2:64,cfg1:64,cfg2:1" timeout 300 python tools/quick_time.py > gpurun_out/r02b_qt_wide.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
cat gpurun_out/r02b_keys.txt gpurun_out/r02b_parity2.txt gpurun_out/r02b_qt.txt gpurun_out/r02b_qt_wide.txt
