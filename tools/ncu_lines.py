"""Per-CUDA-source-line stall samples of an ncu report (--import-source on).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    path, rows, hdr = None, [], None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].rsplit("/", 1)[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0]:  # a source line row (SASS rows have an empty first field)
            d = dict(zip(hdr[2:], r[2:]))
            try:
                samp = int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
                inst = int(d.get("Instructions Executed", 0) or 0)
            except ValueError:
                continue
            rows.append((samp, inst, f"{path}:{r[0]}", r[1].strip()[:80]))
    tot = sum(s for s, *_ in rows) or 1
    print(f"total samples {tot}")
    for s, i, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * s / tot:6.2f}%  {i:>12}  {loc:<22} {src}")


if __name__ == "__main__":
    main()
