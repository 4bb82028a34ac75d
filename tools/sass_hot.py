"""Executed hot set of a kernel: an ncu SASS source page (--page source --csv
--print-source sass) zipped, instruction by instruction, with the kernel's
`nvdisasm -gi` listing (same order), so stall samples and executed instructions
are charged to source lines and to functions on the inlined-at chain.
usage: python tools/sass_hot.py all.txt <kernel-substring> sass.csv [N]   (runs here, no GPU)"""
import collections
import csv
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_size import name_of, spans  # noqa: E402


def listing(path, kern):
    pat = re.compile(r'//## File "([^"]+)", line (\d+)')
    out, loc, fresh, inside = [], [], True, False
    for l in open(path):
        if l.startswith("//---------------------"):
            inside = ".text." in l and kern in l
            continue
        if not inside:
            continue
        m = pat.search(l)
        if m:
            if fresh:
                loc = []
            loc.append((os.path.basename(m.group(1)), int(m.group(2))))
            fresh = False
            continue
        fresh = True
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            out.append(list(loc))
    return out


def main():
    lst, kern, page = sys.argv[1], sys.argv[2], sys.argv[3]
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    locs = listing(lst, kern)
    rows = [r for r in csv.reader(open(page)) if r and r[0].startswith("0x")]
    assert len(rows) == len(locs), (len(rows), len(locs))
    sp = spans()
    smp_line, inst_line = collections.Counter(), collections.Counter()
    smp_fn, inst_fn = collections.Counter(), collections.Counter()
    T = I = 0
    for loc, r in zip(locs, rows):
        s, i = int(r[4]), int(r[5])
        T += s
        I += i
        if not loc:
            continue
        smp_line[loc[0]] += s
        inst_line[loc[0]] += i
        seen = set()
        for f, ln in loc:
            n = name_of(sp, f, ln)
            if n not in seen:
                seen.add(n)
                smp_fn[n] += s
                inst_fn[n] += i
    print("samples %d, warp instructions %d" % (T, I))
    print("-- functions (inclusive of inlined callees)")
    for n, s in smp_fn.most_common(N):
        print("%5.1f%% smp %5.1f%% inst  %s" % (100 * s / T, 100 * inst_fn[n] / I, n))
    src = {}
    base = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_2405_05465_b200", "csrc")
    print("-- source lines (innermost)")
    for (f, ln), s in smp_line.most_common(N):
        if f not in src:
            p = os.path.join(base, f)
            src[f] = open(p).read().split("\n") if os.path.exists(p) else []
        t = src[f][ln - 1].strip()[:70] if 0 < ln <= len(src[f]) else ""
        print("%5.1f%% smp %5.1f%% inst  %s:%d  %s" % (100 * s / T, 100 * inst_line[(f, ln)] / I, f, ln, t))


if __name__ == "__main__":
    main()
