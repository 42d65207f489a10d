"""Join an ncu SASS source export with nvdisasm -g line info: samples / executed per source line.
usage: ncu_lines.py src.csv sim_g.sass [kernel-substring] [N]"""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ia = hdr.index('Address'); iss = hdr.index('Warp Stall Sampling (All Samples)')
iex = hdr.index('Instructions Executed')
kern = sys.argv[3] if len(sys.argv) > 3 else 'sim_kernel'
N = int(sys.argv[4]) if len(sys.argv) > 4 else 50
base = int(data[0][ia], 16)
line_of = {}
insec = False; cur = None
for l in open(sys.argv[2]):
    if l.startswith('.text.'):
        insec = kern in l; continue
    if not insec: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.match(r'^\s+/\*([0-9a-f]+)\*/', l)
    if m: line_of[int(m.group(1), 16)] = cur
S = collections.Counter(); E = collections.Counter()
tot = 0
for d in data:
    o = int(d[ia], 16) - base
    k = line_of.get(o, ('?', 0))
    s = int(d[iss] or 0); e = int(d[iex] or 0)
    S[k] += s; E[k] += e; tot += s
src = {}
for fn in set(f for f, _ in S):
    try:
        src[fn] = open('paper_2504_20828_b200/csrc/' + fn).read().split('\n')
    except OSError:
        src[fn] = []
print(f"total samples {tot}")
for k, s in S.most_common(N):
    f, ln = k
    txt = src.get(f, [])[ln - 1].strip()[:70] if f in src and 0 < ln <= len(src[f]) else ''
    print(f"{s/tot*100:5.2f}% {E[k]:>13,} {f}:{ln:<5} {txt}")
