"""Summarise an ncu report (run here, no GPU needed) into a small text file for profiles/.

    python scripts/ncu_summary.py gpurun_out/k_r01d.ncu-rep > profiles/r01/ncu_kernels.txt

Per kernel: duration, IPC, issued instructions, occupancy, DRAM bytes/throughput, the warp-stall
breakdown (SASS samples) and the instruction share per source function (kernels.cuh).
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issued Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Active Warps per SM",
        "Achieved Active Warps Per SM", "No Eligible", "Compute (SM) Throughput", "DRAM Throughput",
        "Memory Throughput", "L2 Hit Rate", "Waves Per SM", "Grid Size", "Block Size"]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def kernels(rep):
    out = run([rep, "--page", "details", "--csv"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ik, iname, ival, iunit, iid = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                                   hdr.index("Metric Unit"), hdr.index("ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[iid], r[ik])
        per.setdefault(key, {})[r[iname]] = (r[ival], r[iunit])
    return per


def raw_metric(rep, kid, names):
    out = run([rep, "--page", "raw", "--csv", "--print-units", "base"])
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[2:]:
        if r[hdr.index("ID")] != kid:
            continue
        for n in names:
            if n in hdr:
                res[n] = r[hdr.index(n)]
    return res


def stalls_and_functions(rep, kname):
    short = re.sub(r"\(.*", "", kname).split("<")[0].split()[-1].split("::")[-1]
    out = run([rep, "-k", f"regex:{short}", "--page", "source", "--csv", "--print-source", "sass"])
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return "", ""
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in rows[2:]:
        for i in cols:
            try:
                tot[hdr[i]] += int(r[i])
            except (ValueError, IndexError):
                pass
    T = sum(tot.values()) or 1
    st = " ".join(f"{k[6:]}={v / T * 100:.1f}%" for k, v in tot.most_common(8))
    return st, short


def main():
    rep = sys.argv[1]
    for (kid, kname), m in kernels(rep).items():
        print(f"== [{kid}] {kname}")
        for k in KEYS:
            if k in m:
                print(f"   {k:34s} {m[k][0]} {m[k][1]}")
        raw = raw_metric(rep, kid, ["dram__bytes_read.sum", "dram__bytes_write.sum"])
        if raw:
            try:
                rd, wr = float(raw.get("dram__bytes_read.sum", 0)), float(raw.get("dram__bytes_write.sum", 0))
                print(f"   {'dram bytes read+write':34s} {rd + wr:.4g} (read {rd:.4g}, write {wr:.4g})")
            except ValueError:
                pass
        st, _ = stalls_and_functions(rep, kname)
        print(f"   stalls: {st}")


if __name__ == "__main__":
    main()
