"""Summarise an ncu source page (cuda,sass CSV): stall mix, top source lines,
per-function shares.  usage: python tools/ncu_lines.py source.csv raw.csv [N]"""
import csv, collections, re, sys
src_csv, raw_csv = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(raw_csv)))
h = rows[0]; d = dict(zip(h, rows[2]))
keys = [k for k in h if 'smsp__pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued')]
tot = sum(float(d[k] or 0) for k in keys)
print("stalls:", ", ".join("%s %.1f%%" % (k.replace('smsp__pcsamp_warps_issue_stalled_', ''), 100 * float(d[k] or 0) / tot)
                         for k in sorted(keys, key=lambda k: -float(d[k] or 0))[:7]))
print("time", d['gpu__time_duration.sum'], "inst", d['smsp__inst_executed.sum'])
cur = line = None
agg = collections.defaultdict(lambda: [0, 0, set()])
for r in csv.reader(open(src_csv)):
    if not r: continue
    if r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
    if r[0] in ('Function Name', 'Line No'): continue
    if r[0] != '': line = int(r[0]); continue
    if r[2] in ('...', '-'): continue
    a = agg[(cur, line)]; a[0] += int(r[4]); a[1] += int(r[7]); a[2].add(r[2])
T = sum(v[0] for v in agg.values()); I = sum(v[1] for v in agg.values())
base = 'paper_2405_05465_b200/csrc/'
src = {}
for f in ['engine.cu', 'engine.cuh', 'glibc_math.h', 'predictor.cuh']:
    src[f] = open(base + f).read().split('\n')
def text(f, l): return src[f][l - 1].strip()[:80] if f in src and 0 < l <= len(src[f]) else ''
for (f, l), (s, i, ad) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print("%5.1f%% smp %5.1f%% inst %4d  %s:%d  %s" % (100 * s / T, 100 * i / I, len(ad), f, l, text(f, l)))
for f in ['engine.cu', 'engine.cuh']:
    lines = src[f]
    starts = [(i + 1, m.group(1)) for i, l in enumerate(lines)
              for m in [re.match(r'^(?:__device__|template|__global__).*?(\w+)\(', l)] if m]
    by = collections.defaultdict(lambda: [0, 0])
    for (ff, l), (s, i, _) in agg.items():
        if ff != f: continue
        name = '?'
        for st, nm in starts:
            if st <= l: name = nm
        by[name][0] += s; by[name][1] += i
    print(f, "; ".join("%s %.1f%%i %.1f%%s" % (k, 100 * v[1] / I, 100 * v[0] / T)
                       for k, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:10]))
pf = collections.defaultdict(lambda: [0, 0])
for (f, l), (s, i, _) in agg.items(): pf[f][0] += s; pf[f][1] += i
print({k: (round(100 * v[0] / T, 1), round(100 * v[1] / I, 1)) for k, v in pf.items()})
