# bench after the cfg4 warm-pass fix
timeout 900 python bench.py > gpurun_out/r02ce_bench.json 2> gpurun_out/r02ce_bench.err
tail -c 3000 gpurun_out/r02ce_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['configs']['cfg4'], d['configs']['cfg1']['frames_per_s'], d['configs']['cfg3']['frames_per_s'], d['clocks'])"
