"""Summarise an `ncu --set full` report into the text form kept under profiles/:
the details page (section | metric | unit | value, rule text trimmed) plus the
top warp-stall reasons and, when captured with -lineinfo/--import-source, the
SASS instruction mix.  usage: ncu_summary.py report.ncu-rep > profiles/rNN_ncu_full_<name>.txt"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, name, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = page(rep, "details")
    h = rows[0]
    kn, sec, met, unit, val = (h.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                    "Metric Value"))
    print(f"kernel: {rows[1][kn]}")
    for r in rows[1:]:
        if r[met]:
            print(f"{r[sec]} | {r[met]} | {r[unit]} | {r[val]}")
    raw = page(rep, "raw")
    if len(raw) > 2:
        hh, vv = raw[0], raw[2]
        stalls = []
        for i, k in enumerate(hh):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(vv[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        print("\nwarp stall samples (share of all samples):")
        for s, k in sorted(stalls, reverse=True)[:8]:
            print(f"  {k:28s} {100 * s / tot:5.1f}%")
    src = page(rep, "source")
    if len(src) > 2 and "Instructions Executed" in src[1]:
        hs = src[1]
        isrc, iex = hs.index("Source"), hs.index("Instructions Executed")
        ops = collections.Counter()
        for r in src[2:]:
            tok = r[isrc].split()
            if not tok:
                continue
            op = tok[1] if tok[0].startswith("@") else tok[0]
            ops[op.split(".")[0]] += int(r[iex] or 0)
        total = sum(ops.values()) or 1
        print(f"\nSASS warp-instructions executed: {total}")
        for op, c in ops.most_common(12):
            print(f"  {op:10s} {100 * c / total:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
