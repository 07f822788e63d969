"""Hot-instruction view of an ncu report's source page (tuning aid)."""
import collections
import csv
import io
import subprocess
import sys


def main(path, kernel_idx=0, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append(cur)
            continue
        if cur is not None:
            cur.append(r)
    data = blocks[kernel_idx]
    hdr, data = data[0], data[1:]
    iS, iE, iSrc = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"),
                    hdr.index("Source"))
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = [hdr.index(c) for c in cols]
    tot_s = sum(int(r[iS] or 0) for r in data)
    tot = collections.Counter()
    for r in data:
        for j, c in zip(idx, cols):
            tot[c] += int(r[j] or 0)
    print("samples", tot_s, "inst", sum(int(r[iE] or 0) for r in data))
    print("reasons:", ", ".join(f"{c[6:]} {100 * v / tot_s:.0f}%" for c, v in tot.most_common(8)))
    order = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:top]
    for i in sorted(order):
        r = data[i]
        st = sorted([(int(r[j] or 0), c[6:]) for j, c in zip(idx, cols)], reverse=True)[:2]
        print(f"{i:6d} {r[iS]:>5s} {r[iE]:>8s}  {r[iSrc][:64]:64s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
