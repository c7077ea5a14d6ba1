"""Per-source-line warp-stall shares from an ncu report (needs -lineinfo + --import-source):
    python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    data, fname, tot = [], "", 0.0
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = {k: j for j, k in enumerate(r) if k not in ("Source",)}
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            smp = float(r[4] or 0)
        except ValueError:
            continue
        if smp:
            tot += smp
            data.append((smp, f"{fname}:{r[0]}", r[1].strip()[:100]))
    data.sort(reverse=True)
    for smp, loc, src in data[:top]:
        print(f"{100 * smp / tot:5.1f}%  {loc:22s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
