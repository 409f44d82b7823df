"""Per-CUDA-line instruction / stall summary from `ncu --page source --csv --print-source sass,cuda`."""
import sys


def main(path, top=25):
    lines = open(path, errors="replace").read().splitlines()
    hi = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    hdr = lines[hi].strip('"').split('","')
    n = len(hdr)
    i_st, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    rows = []
    for l in lines[hi + 1:]:
        f = l.strip().strip('"').split('","')
        if not f or not f[0].isdigit():
            continue
        src = '","'.join(f[1:len(f) - (n - 2)])
        tail = f[len(f) - (n - 2):]
        try:
            st = float(tail[i_st - 2] or 0)
            ex = float(tail[i_ex - 2] or 0)
        except ValueError:
            continue
        rows.append((int(f[0]), src, st, ex))
    ts = sum(r[2] for r in rows) or 1
    te = sum(r[3] for r in rows) or 1
    print("total executed %.3e warp-instr, %d stall samples" % (te, ts))
    for ln, src, st, ex in sorted(rows, key=lambda r: -r[2])[:top]:
        print("L%4d stall %5.1f%% instr %5.1f%%  %s" % (ln, 100 * st / ts, 100 * ex / te, src.strip()[:90]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
