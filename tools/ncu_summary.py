"""Summarise an ncu report of one kernel: headline metrics, stall mix, and the
hot SASS lines (python tools/ncu_summary.py gpurun_out/x.ncu-rep [--hot N])."""
import collections
import csv
import io
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    hot = int(sys.argv[sys.argv.index("--hot") + 1]) if "--hot" in sys.argv else 25
    rows = ncu_csv(rep, "--page", "details")
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Registers Per Thread",
            "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Executed Instructions", "L2 Hit Rate",
            "L1/TEX Hit Rate"]
    for r in rows[1:]:
        if r[ix["Metric Name"]] in want:
            print(f"{r[ix['Metric Name']]:32s} {r[ix['Metric Value']]:>16s} {r[ix['Metric Unit']]}")
    raw = ncu_csv(rep, "--page", "raw")
    h, v = raw[0], raw[2]
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed_op_local_ld.sum",
              "smsp__inst_executed_op_local_st.sum"]:
        if k in h:
            print(f"{k:60s} {v[h.index(k)]} {raw[1][h.index(k)]}")
    st = [(h[i], float(v[i].replace(",", ""))) for i in range(len(h))
          if "pcsamp_warps_issue_stalled" in h[i] and "not_issued" not in h[i] and v[i].replace(",", "").replace(".", "").isdigit()]
    tot = sum(x for _, x in st) or 1
    print("stalls:", ", ".join(f"{k.split('stalled_')[1]}={x / tot * 100:.1f}%" for k, x in sorted(st, key=lambda t: -t[1])[:10]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = src[1]
    ix = {k: i for i, k in enumerate(h)}
    data = src[2:]
    S = ix["Warp Stall Sampling (All Samples)"]
    E = ix["Instructions Executed"]
    tot = sum(float(r[S] or 0) for r in data) or 1
    bands = collections.Counter()
    mx = max(float(r[E] or 0) for r in data)
    for r in data:
        ex = float(r[E] or 0)
        b = "hot(>=0.8max)" if ex >= 0.8 * mx else ("mid(>=0.1max)" if ex >= 0.1 * mx else "cold")
        bands[b] += float(r[S] or 0)
    print("sample share by exec band:", {k: f"{x / tot * 100:.1f}%" for k, x in bands.items()})
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    top = sorted(range(len(data)), key=lambda i: -float(data[i][S] or 0))[:hot]
    for i in sorted(top):
        r = data[i]
        smp = float(r[S] or 0)
        why = ", ".join(f"{c[6:]}={float(r[ix[c]] or 0) / tot * 100:.1f}" for c in cols if float(r[ix[c]] or 0) / tot * 100 >= 0.2)
        print(f"{i:6d} {smp / tot * 100:5.2f}% ex={float(r[E] or 0) / 1e3:9.1f}k  {r[ix['Source']].strip()[:64]:64s} {why}")


if __name__ == "__main__":
    main()
