"""Static SASS loop summary (profiling aid): for every backward branch of a
kernel, the loop body's instruction count and its DFMA / LDS / IMAD counts.
    cuobjdump -sass lib.so | python tools/sass_loops.py KERNEL_SUBSTRING"""
import re
import sys

pat = sys.argv[1]
lines = sys.stdin.read().split("\n")
funcs, cur = {}, None
for ln in lines:
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if cur and m:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for name, ins in funcs.items():
    if pat not in name:
        continue
    print("==", name[-60:], len(ins), "instructions")
    addr = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA(?:\.U)?(?:\.ANY)?\s+(?:!?P\d,\s*)?0x([0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in addr:
                body = [x for _, x in ins[addr[tgt]: i + 1]]
                cnt = lambda k: sum(1 for x in body if re.search(k, x))
                if cnt(r"\bDFMA\b") == 0:
                    continue
                print(f"  loop {tgt:#06x}-{a:#06x}: {len(body):4d} instr, DFMA {cnt(r'DFMA'):3d}, LDS {cnt(r'LDS'):3d}, "
                      f"IMAD/IADD {cnt(r'IMAD|IADD|LEA'):3d}, UMOV {cnt(r'UMOV'):2d} -> {len(body) / max(1, cnt(r'DFMA')):.2f}/DFMA")
