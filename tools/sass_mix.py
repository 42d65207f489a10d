"""Instruction mix per device function of a disassembled cubin (nvdisasm -c output)."""
import re, sys, collections
lines = open(sys.argv[1]).read().split('\n')
want = sys.argv[2:] or None
cur = None
stats = collections.defaultdict(collections.Counter)
for l in lines:
    m = re.match(r'^([$_]\S+):$', l)
    if m:
        nm = m.group(1)
        mm = re.findall(r'\d+([a-z_][a-z_0-9]*?)E(?:RK|v|N|i|l)', nm)
        cur = mm[-1] if mm else nm[:40]
    m = re.match(r'^\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)', l)
    if m and cur:
        stats[cur][m.group(2).split('.')[0]] += 1
for k, v in sorted(stats.items(), key=lambda kv: -sum(kv[1].values())):
    if want and not any(k.endswith(w) for w in want):
        continue
    print(f"{k[-28:]:>28} {sum(v.values()):6d}", ' '.join(f"{a}:{b}" for a, b in v.most_common(16)))
