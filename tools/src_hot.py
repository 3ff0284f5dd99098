"""Top SASS lines by warp-stall samples from `ncu --page source --csv
--print-source sass` (one or more kernels per file).
usage: python tools/src_hot.py src.csv [top_n] [kernel_substring]"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    want = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = list(csv.reader(open(path)))
    i = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "Kernel Name":
            name = r[1]
            hdr = rows[i + 1]
            j = i + 2
            body = []
            while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
                body.append(rows[j])
                j += 1
            i = j
            if want and want not in name:
                continue
            cs = hdr.index("Warp Stall Sampling (All Samples)")
            ce = hdr.index("Instructions Executed")
            tot = sum(float(b[cs] or 0) for b in body)
            print(f"== {name[:110]}  samples={tot:.0f}")
            body.sort(key=lambda b: -float(b[cs] or 0))
            for b in body[:top]:
                print(f"{float(b[cs] or 0) / tot * 100:5.1f}%  {b[0][-5:]}  {b[1].strip()[:70]:70s} exec={b[ce]}")
        else:
            i += 1


if __name__ == "__main__":
    main()
