"""Instruction mix of the PCG iteration loop of a kernel in libmlmcp.so
(the innermost loop containing the block-reduction butterfly)."""
import collections, re, subprocess, sys
pat = sys.argv[1] if len(sys.argv) > 1 else r"small_propagate_kernel.*GridOp.*Li2E"
txt = subprocess.run(["cuobjdump", "-sass", "paper_2507_19246_b200/libmlmcp.so"],
                     capture_output=True, text=True).stdout
for f in re.split(r'\n\s+Function : ', txt):
    name = f.split('\n')[0]
    if not re.search(pat, name):
        continue
    ins = []
    for l in f.splitlines():
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    loops = []
    for i, (a, t) in enumerate(ins):
        m = re.search(r'BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)', t)
        if m and int(m.group(1), 16) < a:
            loops.append((int(m.group(1), 16), a, i - addr.get(int(m.group(1), 16), 0)))
    for (s, e, n) in sorted(loops, key=lambda x: x[2]):
        body = [t for a, t in ins if s <= a <= e]
        if any('SHFL.BFLY' in t for t in body) and 60 < len(body) < 400:
            c = collections.Counter((t.split()[1] if t.startswith('@') else t.split()[0]).split('.')[0]
                                    for t in body)
            print(name[:70], "loop instructions:", len(body))
            print(c.most_common(20))
            break
