"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[r[ui]]
        name = r[ki].split("(")[0].split("::")[-1]
        out.append((name, v))
    return out


def summary(path, busy_us=5.0):
    launches = load(path)
    agg = collections.defaultdict(list)
    for name, v in launches:
        agg[name].append(v)
    tot = sum(v for _, v in launches)
    lines = ["%-34s %6s %10s %6s %9s %9s %6s" % ("kernel", "n", "total_ms", "share", "median_us", "max_us", "busy")]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        s = sorted(v)
        lines.append("%-34s %6d %10.2f %5.1f%% %9.1f %9.1f %6d" % (
            k[:34], len(v), sum(v) / 1e3, 100 * sum(v) / tot, s[len(s) // 2], s[-1], sum(1 for x in v if x > busy_us)))
    lines.append("total %.2f ms over %d launches" % (tot / 1e3, len(launches)))
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
