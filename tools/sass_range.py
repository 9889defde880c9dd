"""Print the SASS of one kernel between two addresses (hex), comments stripped.
  python tools/sass_range.py lib.so kernel-regex 0xLO 0xHI"""
import re, subprocess, sys
lib, kre, lo, hi = sys.argv[1], re.compile(sys.argv[2]), int(sys.argv[3], 16), int(sys.argv[4], 16)
cur = None
for line in subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if cur and kre.search(cur) and m and lo <= int(m.group(1), 16) <= hi:
        print(f"{m.group(1)}  {m.group(2).strip()}")
