"""Static instruction mix of a kernel's hottest loop from cuobjdump SASS:
python tools/sass_loop.py LIB_OR_CUBIN MANGLED_NAME_SUBSTRING [ANCHOR=SHFL.DOWN]
The loop is the range [target, branch] of the first backward branch after
the first ANCHOR instruction; rare out-of-line paths inside it are counted."""
import collections
import re
import subprocess
import sys

path, name = sys.argv[1], sys.argv[2]
anchor = sys.argv[3] if len(sys.argv) > 3 else "SHFL.DOWN"
sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
funcs = sass.split("Function : ")
body = next(f for f in funcs if f.startswith(name) or name in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
a = next(i for i, (_, t) in enumerate(ins) if anchor in t)
for j in range(a, len(ins)):
    m = re.search(r"BRA (?:`\(.*?\))?\s*0x([0-9a-f]+)", ins[j][1])
    if m and int(m.group(1), 16) < ins[j][0]:
        lo = int(m.group(1), 16)
        break
loop = [t for addr, t in ins if lo <= addr <= ins[j][0]]
ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in loop)
print(f"loop 0x{lo:x}-0x{ins[j][0]:x}: {len(loop)} instructions")
for op, n in ops.most_common():
    print(f"  {op:24s} {n}")
