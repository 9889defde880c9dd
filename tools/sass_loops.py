"""Static SASS check for the issue-bound kernels: for every loop (backward
branch) of the selected kernels, its instruction count and opcode histogram.
Used to A/B kernel variants here (no GPU) before spending GPU time: K3 is
issue-bound, so instructions per loop trip track its time.

  python tools/sass_loops.py [lib.so] [kernel-regex] [min-loop-size]
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2112_13169_b200/lib/libvxm.so"
kre = re.compile(sys.argv[2] if len(sys.argv) > 2 else "trace_bundle")
min_size = int(sys.argv[3]) if len(sys.argv) > 3 else 40

sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs, cur = {}, None
ins = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur is None:
        continue
    m = ins.search(line)
    if m:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))

for name, body in funcs.items():
    if not kre.search(name):
        continue
    addr = {a: i for i, (a, _) in enumerate(body)}
    print(f"== {name}: {len(body)} instructions, "
          f"{sum(1 for _, t in body if t.split()[0] in ('STL', 'LDL') or ' STL' in t or ' LDL' in t)} local-memory ops")
    for i, (a, text) in enumerate(body):
        m = re.search(r"BRA\s+(?:P\d,\s*)?(?:!?P\d,\s*)?(0x[0-9a-f]+)", text)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr:
            continue
        lo = addr[tgt]
        loop = body[lo:i + 1]
        if len(loop) < min_size:
            continue
        ops = collections.Counter()
        for _, t in loop:
            t = re.sub(r"^@!?U?P\w+\s+", "", t)
            ops[t.split()[0].split(".")[0]] += 1
        top = ", ".join(f"{k} {v}" for k, v in ops.most_common(18))
        print(f"  loop 0x{tgt:x}-0x{a:x}: {len(loop)} instr  [{top}]")
