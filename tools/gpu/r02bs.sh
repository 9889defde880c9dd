# compute-sanitizer over the round-2 kernels incl. the chain merges with in-kernel publish
timeout 1500 bash tools/sanitize.sh > gpurun_out/r02bs_sanitize.log 2>&1
for f in gpurun_out/sanitizer_*.txt; do cp $f ${f/sanitizer_/r02bs_sanitizer_}; done
tail -n 3 gpurun_out/r02bs_sanitizer_*.txt
