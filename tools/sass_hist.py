#!/usr/bin/env python
"""Per-kernel SASS opcode histogram of a cubin / .so (cuobjdump -sass), with a rough
fma-heavy pipe cycle estimate (IMAD.WIDE / IMAD.HI count 4 cycles per warp, other IMAD 2).
usage: sass_hist.py <file> <kernel-name-substring> [top]"""
import re, subprocess, sys, collections
f, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["cuobjdump", "-sass", f], capture_output=True, text=True).stdout
fn = None
hist = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1); continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if m and fn:
        hist[fn][m.group(1)] += 1
for fn, h in hist.items():
    if pat not in fn: continue
    tot = sum(h.values())
    wide = sum(v for k, v in h.items() if k.startswith("IMAD.WIDE") or k.startswith("IMAD.HI"))
    imad = sum(v for k, v in h.items() if k.startswith("IMAD")) - wide
    alu = sum(v for k, v in h.items() if re.match(r"(IADD3|LOP3|SEL|ISETP|SHF|LEA|MOV|PRMT|VIADD|IMNMX|VIMNMX)", k))
    print(f"== {fn}: {tot} instr; wide/hi {wide}, other IMAD {imad} -> fma cycles {4*wide+2*imad}; alu-ish {alu}")
    print("   " + ", ".join(f"{k} {v}" for k, v in h.most_common(top)))
