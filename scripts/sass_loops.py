"""Loops of one kernel's SASS (cuobjdump -sass): backward branches, their body size and
opcode mix, for loops containing a given opcode.  usage: sass_loops.py FILE.sass [OPCODE]"""
import re, sys, collections
ins = []
for l in open(sys.argv[1]):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
want = sys.argv[2] if len(sys.argv) > 2 else "FFMA"
def op(s):
    t = s.split()
    if t[0].startswith("@"): t = t[1:]
    return t[0]
for a, s in ins:
    if op(s).startswith("BRA"):
        m = re.search(r"0x([0-9a-f]+)\s*$", s)
        if m and int(m.group(1), 16) < a:
            lo = int(m.group(1), 16)
            body = [op(x) for b, x in ins if lo <= b <= a]
            c = collections.Counter(o.split(".")[0] for o in body)
            if c[want]:
                print(f"loop {lo:#x}-{a:#x}: {len(body)} instrs, {c[want]} {want}; " +
                      ", ".join(f"{k} {v}" for k, v in c.most_common(14)))
