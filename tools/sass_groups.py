import re, sys
lines = open(sys.argv[1]).read().split('\n')
sass = [l for l in lines if re.match(r'\s*\d+\.\d+% thr=', l)]
groups = []
for l in sass:
    m = re.match(r'\s*(\d+\.\d+)% thr=\s*(\d+) smp=\s*(\d+) (.*)', l)
    sh, thr, smp, ins = float(m.group(1)), int(m.group(2)), int(m.group(3)), m.group(4)
    if groups and abs(groups[-1]['sh'] - sh) < 0.006 and groups[-1]['thr'] == thr:
        g = groups[-1]; g['n'] += 1; g['smp'] += smp; g['tot'] += sh; g['ins'].append(ins)
    else:
        groups.append(dict(sh=sh, thr=thr, n=1, smp=smp, tot=sh, ins=[ins]))
tots = sum(g['smp'] for g in groups)
thresh = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
for g in groups:
    if g['tot'] > thresh:
        mem = [(i.split()[0] if not i.startswith('@') else i.split()[1]) for i in g['ins'] if any(k in i for k in ('LDG', 'LDS', 'STS', 'LDL', 'STL', 'ATOM', 'SHFL', 'VOTE', 'LD.E', 'ST.E', 'STG', 'I2F', 'MUFU', 'WARPSYNC'))]
        print(f"share {g['tot']:6.2f}%  n={g['n']:3d} thr={g['thr']:2d} samples {g['smp'] / tots * 100:5.1f}%  first: {g['ins'][0][:44]:44s} | {' '.join(mem)[:120]}")
