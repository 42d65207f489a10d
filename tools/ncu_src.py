"""Per-function / per-instruction view of an ncu source export (--page source --csv --print-source sass).
usage: ncu_src.py src.csv sim.sass [function-suffix [N]]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ia = hdr.index('Address'); isrc = hdr.index('Source')
iss = hdr.index('Warp Stall Sampling (All Samples)'); iex = hdr.index('Instructions Executed')
base = int(data[0][ia], 16)
funcs = []; insec = False
for l in open(sys.argv[2]).read().split('\n'):
    if l.startswith('.text.'):
        insec = 'sim_kernel' in l
        continue
    if not insec:
        continue
    m = re.match(r'^([$_]\S+):$', l)
    if m:
        nm = m.group(1); mm = re.findall(r'\d+([a-z_][a-z_0-9]*?)E(?:RK|v|N|i|l)', nm)
        funcs.append([(mm[-1] if mm else nm[-30:]), None])
    m = re.match(r'^\s+/\*([0-9a-f]+)\*/\s+(.*)', l)
    if m and funcs and funcs[-1][1] is None:
        funcs[-1][1] = int(m.group(1), 16)
funcs = sorted([(a, b) for a, b in funcs if b is not None], key=lambda x: x[1])
def fn(o):
    r = 'body'
    for a, b in funcs:
        if b <= o:
            r = a
    return r
want = sys.argv[3] if len(sys.argv) > 3 else None
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
sel = []
for d in data:
    o = int(d[ia], 16) - base
    f = fn(o)
    if want and not f.endswith(want):
        continue
    sel.append((o, int(d[iss] or 0), int(d[iex] or 0), d[isrc].strip()))
tot = sum(s for _, s, _, _ in sel)
ex = sum(e for _, _, e, _ in sel)
print(f"samples {tot} executed {ex:,}")
if len(sys.argv) > 5:   # listing in address order of executed instructions
    for o, s, e, t in sel:
        if e:
            print(f"{o:6x} {s:7d} {e:13,} {t[:90]}")
else:
    for o, s, e, t in sorted(sel, key=lambda x: -x[1])[:N]:
        print(f"{o:6x} {s:7d} {e:13,} {t[:90]}")
