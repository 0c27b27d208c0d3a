"""Stall samples per CUDA source line from an ncu report (needs -lineinfo and
--import-source on):  python tools/srcline.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, res = None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0].isdigit() and len(r) > 7 and r[2] == "-":
            s = int(r[4]) if r[4] not in ("-", "") else 0
            e = int(r[7]) if r[7] not in ("-", "") else 0
            res.append((s, e, fname, int(r[0]), r[1].strip()[:80]))
    tot = sum(x[0] for x in res) or 1
    res.sort(reverse=True)
    for s, e, f, line, text in res[:top]:
        print(f"{100 * s / tot:5.1f}% {e / 1e6:9.1f}M {f}:{line} {text}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
