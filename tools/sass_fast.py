"""Instructions of the batch ray cast's fast chunk (VOTE.ALL .. the branch
back to the loop head) and its exact chunk, for A/B builds (static count).
  python tools/sass_fast.py [lib.so] [kernel-regex]"""
import collections, re, subprocess, sys
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2112_13169_b200/lib/libvxm.so"
kre = re.compile(sys.argv[2] if len(sys.argv) > 2 else "ILi4ELi2E")
body, cur = [], None
for line in subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if cur and kre.search(cur) and m:
        body.append((int(m.group(1), 16), m.group(2).strip()))
idx = {a: i for i, (a, _) in enumerate(body)}
# the in-grid loop: the VOTE.ALL of the fast test
va = [i for i, (_, t) in enumerate(body) if "VOTE.ALL" in t]
for v in va:
    # loop head: the backward branch target that encloses v
    heads = []
    for i, (a, t) in enumerate(body):
        m = re.search(r"BRA\s+(?:!?U?P\d,\s*)?(0x[0-9a-f]+)", t)
        if m and i > v and int(m.group(1), 16) < body[v][0]:
            heads.append((i, idx.get(int(m.group(1), 16))))
    if not heads:
        continue
    tail, head = min(heads)
    # the exact chunk: the target of the branch right after VOTE.ALL
    m = re.search(r"BRA\s+(0x[0-9a-f]+)", body[v + 2][1] if "BRA" in body[v + 2][1] else body[v + 1][1])
    ex = idx[int(m.group(1), 16)] if m else None
    def hist(lo, hi):
        c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t in body[lo:hi])
        return ", ".join(f"{k} {n}" for k, n in c.most_common(14))
    print(f"head+test: {v - head + 1}   fast chunk: {ex - v - 1 if ex else '?'}   exact chunk: {tail - ex + 1 if ex else '?'}")
    if ex:
        print("  fast :", hist(v + 1, ex))
        print("  exact:", hist(ex, tail + 1))
    ll = sum(1 for _, t in body[head:tail + 1] if re.search(r"\b(LDL|STL)\b", t))
    print("  local-memory ops in the loop:", ll)
