"""List the big loops (backward branches) of a kernel's SASS with op counts.
usage: python tools/sass_loops.py LIB.so MANGLED_KERNEL_NAME [min_len]"""
import re, subprocess, sys, collections
lib, fn = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 200
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for l in out.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
print("total instructions", len(ins))
for a, t in ins:
    m = re.search(r"BRA\s.*?(0x[0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt < a and (a - tgt) // 16 >= minlen:
            body = [x for x in ins if tgt <= x[0] <= a]
            c = collections.Counter(x[1].split()[0].lstrip("@!P0123456789 ") for x in body)
            print(hex(tgt), hex(a), len(body), dict(c.most_common(12)))
