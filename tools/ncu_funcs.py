"""Executed instructions and stall samples per device function of one kernel: joins an ncu SASS
source export with `nvdisasm -c` output.  usage: ncu_funcs.py src.csv kernel.sass section-substring"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows[:5]) if 'Address' in r)
h = rows[hi]; data = rows[hi + 1:]
ia, iex, iss = h.index('Address'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
base = int(data[0][ia], 16)
funcs = []; insec = False
for l in open(sys.argv[2]):
    l = l.rstrip('\n')
    if l.startswith('.text.'):
        insec = sys.argv[3] in l
        if insec: funcs.append(('kernel', 0))
        continue
    if not insec: continue
    m = re.match(r'^([$_.]?\S+):$', l)
    if m and not l.startswith('.L'):
        nm = m.group(1); mm = re.findall(r'\d+([a-z_][a-z_0-9]*?)E(?:RK|v|N|i|l)', nm)
        funcs.append([(mm[-1] if mm else nm[-40:]), None])
    m = re.match(r'^\s+/\*([0-9a-f]+)\*/\s+(.*)', l)
    if m and funcs and funcs[-1][1] is None:
        funcs[-1][1] = int(m.group(1), 16)
funcs = sorted([(a, b) for a, b in funcs if b is not None], key=lambda x: x[1])
ex = collections.Counter(); st = collections.Counter(); sz = collections.Counter()
for d in data:
    o = int(d[ia], 16) - base
    f = 'kernel'
    for a, b in funcs:
        if b <= o: f = a
    ex[f] += int(d[iex] or 0); st[f] += int(d[iss] or 0); sz[f] += 16
te, ts = sum(ex.values()), sum(st.values())
for f, e in ex.most_common(25):
    print(f"{f[:34]:34s} {e/te*100:6.1f}% inst {st[f]/ts*100:6.1f}% stalls  {sz[f]:7d} B")
