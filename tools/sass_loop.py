"""Opcode histogram of the body of the first backward branch loop whose body contains FADD2.

usage: python tools/sass_loop.py file.sass   (cuobjdump -sass output of one function)
"""
import collections
import re
import sys

L = open(sys.argv[1]).read().splitlines()
addr = {}
for i, l in enumerate(L):
    m = re.match(r'\s+/\*([0-9a-f]+)\*/', l)
    if m:
        addr[int(m.group(1), 16)] = i
for i, l in enumerate(L):
    m = re.search(r'BRA(\.U)? [^,]*?,? ?0x([0-9a-f]+)', l)
    if not m:
        continue
    tgt = int(m.group(2), 16)
    here = re.match(r'\s+/\*([0-9a-f]+)\*/', l)
    if here and tgt < int(here.group(1), 16) and tgt in addr:
        body = L[addr[tgt]:i + 1]
        if not any('FADD2' in b for b in body):
            continue
        c = collections.Counter()
        for b in body:
            mm = re.match(r'\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?([A-Z0-9_]+)', b)
            if mm:
                c[mm.group(2)] += 1
        print(f"loop {tgt:#x}..{here.group(1)}: {sum(c.values())} instructions")
        print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
        break
