"""Print the SASS of one kernel of libwhff_b200.so (static instruction mix).
Usage: python tools/sass_fn.py <mangled-name-substring> [--mix]"""
import collections
import re
import subprocess
import sys

lib = "paper_1902_08018_b200/libwhff_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
want = sys.argv[1]
cur, lines = None, []
for ln in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    if cur == want and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(ln)
if "--mix" in sys.argv:
    mix = collections.Counter()
    for ln in lines:
        ins = re.sub(r"^\s+/\*[0-9a-f]+\*/\s+", "", ln)
        ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
        mix[ins.split()[0].split(".")[0]] += 1
    print(len(lines), "instructions")
    for k, v in mix.most_common(30):
        print(f"{v:6d} {k}")
else:
    print("\n".join(lines))
