"""Summarise a coarse_cl GROUP/REPLAY trace (ISMG_CL_TRACE build): time per group size."""
import collections, re, sys

dmax = int(sys.argv[2]) if len(sys.argv) > 2 else 381
d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r'(GROUP|REPLAY) G=(\d+) ns=(\d+)', line)
    if m:
        d[(m[1], int(m[2]))].append(int(m[3]))
tot = 0
for k in sorted(d):
    v = d[k]
    steps = dmax + 8 * (k[1] - 1) + (5 if k[0] == 'GROUP' else 1)
    tot += sum(v)
    print("%-6s G=%-4d n=%-4d mean %8.1f us  %5.0f ns/step  total %6.1f ms"
          % (k[0], k[1], len(v), sum(v) / len(v) / 1e3, sum(v) / len(v) / steps, sum(v) / 1e6))
print("total group ms %.1f" % (tot / 1e6))
