"""Per-unit phase split of the longest units of each sweep launch (diagnostic).

Reads an SSG_DUMP_UNITS file written by a -DSSG_PHASE_CYCLES build
(engine.cuh SSG_PH_*): P lines carry the phase cycles, plain lines the unit
(config shape, iterations, cycles)."""
import sys

P, U = {}, {}
for l in open(sys.argv[1]):
    p = l.split()
    if p[0] == "P":
        P[(int(p[1]), int(p[2]))] = list(map(int, p[3:]))
        continue
    if p[0] == "#":
        continue
    k = (int(p[0]), int(p[1]))
    U[k] = dict(n=int(p[3]), it=int(p[5]), cyc=int(p[6]), pol=int(p[8]), mb=int(p[9]),
                ent=int(p[10]), tp=int(p[11]), pp=int(p[12]), chunk=int(p[13]))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 3
for L in sorted({k[0] for k in U}):
    for k in sorted([k for k in U if k[0] == L], key=lambda k: -U[k]["cyc"])[:top]:
        u, ph = U[k], P.get(k)
        if not ph:
            continue
        nff = max(1, u["it"] - ph[5])
        print("L%d pol%d tp%d pp%d mb%d it %d ent/it %.1f | ff it %d calls %d (%.1f/call, %.0f cyc/call) |"
              " normal it: sched %.0f lat %.0f (sums %.0f query %.0f ops %.0f makespan %.0f) compl %.0f cyc |"
              " arrivals %.0f%% | total %.0fM cyc | >32 runners %d, queue+room %d, ff empty %d, prefill batches %d"
              % (L, u["pol"], u["tp"], u["pp"], u["mb"], u["it"], u["ent"] / max(1, u["it"]), ph[5], ph[7],
                 ph[5] / max(1, ph[7]), ph[3] / max(1, ph[7]), ph[0] / nff, ph[1] / nff,
                 ph[8] / nff, ph[9] / nff, ph[11] / nff, ph[10] / nff, ph[2] / nff,
                 100.0 * ph[4] / ph[6], ph[6] / 1e6, ph[12], ph[13], ph[14], ph[15]))
