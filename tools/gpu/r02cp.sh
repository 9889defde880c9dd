# randomised parity sweeps at the final state (after K3 lone tail-fast and K4 coordinates)
timeout 1100 python tools/fuzz_parity.py 900 801 > gpurun_out/r02cp_fuzz_parity.txt 2>&1; echo "parity rc $?"
timeout 500 python tools/fuzz_stages.py 300 802 > gpurun_out/r02cp_fuzz_stages.txt 2>&1; echo "stages rc $?"
tail -n 1 gpurun_out/r02cp_fuzz_parity.txt gpurun_out/r02cp_fuzz_stages.txt
grep -c "aligned': True" gpurun_out/r02cp_fuzz_parity.txt
