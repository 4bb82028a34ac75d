"""SASS size of a kernel attributed to source functions (I-cache budget work).

    cuobjdump -xelf all build/ssg/engine.o   (in a scratch dir)
    nvdisasm -gi engine.sm_100a.cubin > all.txt
    python tools/sass_size.py all.txt <kernel-substring> [--chain]

Each instruction is charged to the innermost source line nvdisasm reports and,
with --chain, to every function on its inlined-at chain (so a helper's total
includes everything inlined into it).  Function spans come from a brace scan of
the csrc sources."""
import collections
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2405_05465_b200", "csrc")
DEF = re.compile(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__|__host__ __device__|static __device__)[^;{]*?\b(\w+)\s*\(")


def spans():
    out = {}
    for fn in os.listdir(CSRC):
        if not fn.endswith((".cu", ".cuh", ".h")):
            continue
        lines = open(os.path.join(CSRC, fn)).read().split("\n")
        cur, depth, start, base = None, 0, 0, 0
        pending = None
        for i, l in enumerate(lines, 1):
            m = DEF.match(l.strip())
            if m and cur is None:
                pending = (m.group(1), i)
            if pending and "{" in l and cur is None:
                cur, start = pending
                base = depth
                pending = None
            depth += l.count("{") - l.count("}")
            if cur and depth == base and "}" in l:
                out.setdefault(fn, []).append((start, i, cur))
                cur = None
    return out


def name_of(sp, f, line):
    base = os.path.basename(f)
    for a, b, n in sp.get(base, []):
        if a <= line <= b:
            return "%s:%s" % (base, n)
    return "%s:?" % base


def main():
    path, kern = sys.argv[1], sys.argv[2]
    chain = "--chain" in sys.argv
    sp = spans()
    inside = False
    loc = []
    tot = 0
    by = collections.Counter()
    pat = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    fresh = True
    for l in open(path):
        if l.startswith("//---------------------"):
            inside = (".text." in l and kern in l)
            continue
        if not inside:
            continue
        m = pat.search(l)
        if m:
            # a group of //## lines precedes each instruction run: the first is
            # the innermost location with its inlined-at chain
            # (each line is one level: "File X line a inlined at Y line b")
            if fresh:
                loc = []
            loc.append((m.group(1), int(m.group(2))))
            fresh = False
            continue
        fresh = True
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            tot += 1
            if not loc:
                continue
            if chain:
                seen = set()
                for f, ln in loc:
                    n = name_of(sp, f, ln)
                    if n not in seen:
                        by[n] += 1
                        seen.add(n)
            else:
                by[name_of(sp, *loc[0])] += 1
    print("total %d instructions (%d KB)" % (tot, tot * 16 // 1024))
    for n, c in by.most_common(60):
        print("%7d %6.1f%%  %s" % (c, 100.0 * c / tot, n))


if __name__ == "__main__":
    main()
