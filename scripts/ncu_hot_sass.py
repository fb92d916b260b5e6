"""Top stalled SASS instructions of each kernel in an ncu report (source page, sass view)."""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    blocks, cur = [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    for blk in blocks:
        name = next(csv.reader([blk[0]]))[1]
        rows = list(csv.reader(blk[1:]))
        hdr = rows[0]
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        data = []
        tot = 0
        for r in rows[1:]:
            try:
                v = int(r[iS])
            except (ValueError, IndexError):
                continue
            tot += v
            reasons = sorted(((int(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:3]
            data.append((v, r[1].strip(), reasons))
        print(f"===== {name}: {tot} samples")
        for v, src, reasons in sorted(data, reverse=True)[:top]:
            rs = ", ".join(f"{h[6:]}={c}" for c, h in reasons if c)
            print(f"{100 * v / max(tot, 1):5.1f}%  {src[:60]:60s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
