set -x
timeout 900 python -m pytest tests/test_gpu_keys.py tests/test_gpu_snapshot.py tests/test_gpu_parity.py tests/test_gpu_sequence.py -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02c_t1.txt
QT_CONFIGS="cfg2:64,cfg1:64,cfg3:16,cfg2:1" timeout 300 python tools/quick_time.py > gpurun_out/r02c_qt.txt 2>&1
QT_FLAGS=64 QT_CONFIGS="cfg2:64,cfg3:16" timeout 300 python tools/quick_time.py > gpurun_out/r02c_qt_clear.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r02c_all.txt
cat gpurun_out/r02c_t1.txt gpurun_out/r02c_qt.txt gpurun_out/r02c_qt_clear.txt gpurun_out/r02c_all.txt
