"""Per-opcode instruction counts and stall samples of one kernel in an ncu report
(run here, no GPU needed):

    python scripts/sass_profile.py gpurun_out/x.ncu-rep [n_warps] [--runs] [--kernel=REGEX]

n_warps normalises counts to per-warp figures; --runs prints the hot straight-line
runs (same execution count) with their stall-sample share.
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    nw = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 1.0
    kf = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--kernel=")]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                         (["-k", "regex:" + kf[0]] if kf else []),
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    # with several kernels in the report only the first section is read (use --kernel=REGEX)
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(hdr):
            data.append(r)
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    smp = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    cnt, samp = collections.Counter(), collections.Counter()
    seq = []
    for r in data:
        n = int(r[ie] or 0)
        toks = r[src].split()
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
        cnt[op] += n
        samp[op] += int(r[smp] or 0)
        seq.append((r, n, int(r[smp] or 0)))
    tot, tsamp = sum(cnt.values()), sum(samp.values())
    print(f"instructions/warp {tot / nw:.0f}  samples {tsamp}")
    for k, v in cnt.most_common(16):
        print(f"  {k:8s} {v / nw:9.1f} {100 * v / tot:5.1f}%  samples {100 * samp[k] / tsamp:5.1f}%")
    if "--runs" in sys.argv:
        runs = []
        for i, (r, n, sm) in enumerate(seq):
            if runs and runs[-1]["n"] == n:
                runs[-1]["len"] += 1
                runs[-1]["s"] += sm
                runs[-1]["rows"].append(r)
            else:
                runs.append({"i": i, "len": 1, "n": n, "s": sm, "rows": [r]})
        for ru in runs:
            if ru["s"] > float(next((a.split("=")[1] for a in sys.argv if a.startswith("--min=")), 0.015)) * tsamp:
                st = collections.Counter()
                for r in ru["rows"]:
                    for c in stall_cols:
                        st[c[6:]] += int(r[hdr.index(c)] or 0)
                top = ", ".join(f"{k}={v}" for k, v in st.most_common(4))
                print(f"  idx {ru['i']:5d} len {ru['len']:4d} x{ru['n'] / nw:6.2f}  {100 * ru['s'] / tsamp:5.1f}%  "
                      f"{ru['rows'][0][src].strip()[:30]:30s} {top}")


if __name__ == "__main__":
    main()
