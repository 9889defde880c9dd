# randomised parity sweeps at HEAD (after the merge4 byte-permute decode and the K2 pack MSB test)
mkdir -p gpurun_out
timeout 1100 python tools/fuzz_parity.py 900 811 > gpurun_out/r02cv_fuzz_parity.txt 2>&1; echo "parity rc $?"
timeout 500 python tools/fuzz_stages.py 300 812 > gpurun_out/r02cv_fuzz_stages.txt 2>&1; echo "stages rc $?"
tail -n 1 gpurun_out/r02cv_fuzz_parity.txt gpurun_out/r02cv_fuzz_stages.txt
grep -c "aligned': True" gpurun_out/r02cv_fuzz_parity.txt
