# randomised parity sweeps at the final round-2 state (aligned corridor cases added to fuzz_parity)
timeout 900 python tools/fuzz_parity.py 700 601 > gpurun_out/r02cd_fuzz_parity.txt 2>&1; echo "parity rc $?"
timeout 500 python tools/fuzz_stages.py 300 602 > gpurun_out/r02cd_fuzz_stages.txt 2>&1; echo "stages rc $?"
tail -n 2 gpurun_out/r02cd_fuzz_parity.txt gpurun_out/r02cd_fuzz_stages.txt
grep -c "aligned': True" gpurun_out/r02cd_fuzz_parity.txt
