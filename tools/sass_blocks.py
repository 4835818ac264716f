"""Group an ncu SASS source-page CSV (ncu -i X --page source --csv --print-source sass) into
basic blocks (runs of equal execution count) and print each block's share of warp
instructions and stall samples -- the per-phase instruction budget of a kernel."""
import csv
import sys


def main(path, min_share=0.2):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    I, S, T = (hdr.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)",
                                      "Avg. Threads Executed"))
    data = [(r[1].strip(), int(r[I]), int(r[S]), float(r[T])) for r in rows[2:] if len(r) > I]
    tot = sum(d[1] for d in data) or 1
    st = sum(d[2] for d in data) or 1
    print(f"total warp instructions {tot}, stall samples {st}")
    i = 0
    while i < len(data):
        j = i
        while j + 1 < len(data) and data[j + 1][1] == data[i][1] and not data[j][0].split()[0].endswith("BRA"):
            j += 1
        blk = data[i:j + 1]
        ins = sum(d[1] for d in blk)
        stl = sum(d[2] for d in blk)
        if ins / tot * 100 >= min_share or stl / st * 100 >= min_share:
            ops = " ".join(d[0].split()[0] if not d[0].startswith("@") else d[0].split()[1] for d in blk)
            print(f"[{i:4d}-{j:4d}] n={len(blk):3d} x{data[i][1]:9d} thr{data[i][3]:5.1f} "
                  f"inst {ins / tot * 100:5.1f}% stall {stl / st * 100:5.1f}%  {ops[:150]}")
        i = j + 1


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.2)
