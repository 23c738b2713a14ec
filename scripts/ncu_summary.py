"""Summaries of the ncu captures for profiles/ (run here on the merged
gpurun_out/ files).

  python scripts/ncu_summary.py full REPORT.ncu-rep OUT.csv TRAFFIC.json "nt n1 n2" [LABEL]
      (merges the per-pass DRAM traffic into TRAFFIC.json under the key "ntxn1xn2")
  python scripts/ncu_summary.py launches LAUNCHES.csv OUT.csv "command"
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

# algorithmic N-vector passes per launch (SURVEY.md 8d / DESIGN.md)
ALG = {"K1_row_p_update_B": 6, "K2_col_S_mid": 4, "K3_row_BT_update": 4, "P1_hartley_x2": 2,
       "P2_hartley_x1": 2, "P3_t_filter": 2, "P4_hartley_x1": 2, "P5_hartley_x2_dot": 3, "X_axpy": 3,
       # BASELINE C1: matvec row (2N) + column-with-accumulate (3N); 2-level solve 3 x 2N
       "row_apply": 2, "col_acc": 3, "C1_pfa_x2": 2, "C1_pfa_x1": 2}


def pass_name(kernel, seen):
    k = kernel.split("(")[0]
    prev = seen.get("prev", "")
    seen["prev"] = k
    if "k_rowq" in k:
        return "K1_row_p_update_B" if ", 2>" in k else "K3_row_BT_update"
    if "k_rowc" in k or "k_row<" in k:
        return "K1_row_p_update_B" if ", 2," in k else ("K3_row_BT_update" if ", 1," in k else "row_apply")
    if "k_colc" in k or "k_col<" in k:
        return "K2_col_S_mid" if ", 2," in k else "col_acc"
    if "k_t_filter" in k:
        return "P3_t_filter"
    if "k_hartley_row" in k:  # P5 follows the second x1 pass, P1 opens the solve
        return "P5_hartley_x2_dot" if "k_hartley_col" in prev else "P1_hartley_x2"
    if "k_hartley_col" in k:
        # P2 follows the x2 pass, P4 the t filter (a capture window may open on P4)
        return "P2_hartley_x1" if "k_hartley_row" in prev else "P4_hartley_x1"
    if "k_axpy_dev" in k:
        return "X_axpy"
    if "k_pfa_hrow" in k:
        return "C1_pfa_x2"
    if "k_pfa_hcol" in k:
        return "C1_pfa_x1"
    return k.replace("void ", "")


def f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def full(rep, out_csv, traffic_json, shape="256 256 256", label="C2"):
    dims = [int(v) for v in shape.split()]
    n_elem = dims[0] * dims[1] * dims[2]
    key = "x".join(str(v) for v in dims)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "second": 1e6, "s": 1e6}

    def g(r, m):
        if m not in ix:
            return float("nan")
        return f(r[ix[m]]) * scale.get(units[ix[m]], 1.0)
    seen, out, traffic, fp64, issue = {}, [], OrderedDict(), OrderedDict(), OrderedDict()
    for r in data:
        name = pass_name(r[ix["Kernel Name"]], seen)
        us = g(r, "gpu__time_duration.sum")
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        alg = ALG.get(name, float("nan")) * 8 * n_elem
        out.append([name, r[ix["Kernel Name"]].split("(")[0].replace("void ", ""), f"{us:.1f}",
                    f"{rd / 1e6:.1f}", f"{wr / 1e6:.1f}", f"{(rd + wr) / 1e6:.1f}", f"{alg / 1e6:.1f}",
                    f"{(rd + wr) / alg:.2f}", f"{(rd + wr) / (us * 1e-6) / 1e9:.0f}",
                    f"{g(r, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.1f}",
                    f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}",
                    f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}",
                    f"{g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f}",
                    f"{g(r, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum') / 1e6:.2f}",
                    f"{g(r, 'launch__registers_per_thread'):.0f}"])
        if name in ALG and name not in traffic:
            traffic[name] = rd + wr
            fp64[name] = round(g(r, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'), 1)
            issue[name] = round(g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'), 1)
    with open(out_csv, "w") as fh:
        fh.write(f"# ncu --set full summary ({label} {key}, kernels of one PCG iteration; {rep.split('/')[-1]})\n")
        fh.write("# traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch; alg = algorithmic bytes\n")
        w = csv.writer(fh)
        w.writerow(["pass", "kernel", "us", "dram_read_MB", "dram_write_MB", "traffic_MB", "alg_MB",
                    "traffic/alg", "dram_GBs", "fp64_pipe_pct", "warps_active_pct", "issue_active_pct",
                    "l1tex_throughput_pct", "smem_wavefronts_M", "regs"])
        w.writerows(out)
    try:
        allcap = json.load(open(traffic_json))
    except Exception:  # noqa: BLE001
        allcap = {}
    allcap[key] = {"source": f"{out_csv} (ncu --set full, {label} {key})", "traffic": traffic,
                   "fp64_pipe_pct": fp64, "issue_active_pct": issue}
    with open(traffic_json, "w") as fh:
        json.dump(allcap, fh, indent=1)
    for row in out:
        print(",".join(row))


def launches(log, out_csv, cmd):
    lines = [l for l in open(log) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = OrderedDict()
    for r in rows[1:]:
        if len(r) != len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("fdg::", "")
        v = f(r[ix["Metric Value"]])
        unit = r[ix["Metric Unit"]]
        v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    with open(out_csv, "w") as fh:
        fh.write("# ncu launch list (gpu__time_duration.sum, --clock-control none)\n")
        fh.write(f"# command: {cmd}\n")
        fh.write("# cold-cache, serialised per-launch times: compare SHARES, not absolutes\n")
        fh.write(f"# total launches {n}, total device time {tot / 1000:.2f} ms\n")
        fh.write("kernel,launches,total_us,share_pct,avg_us\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k},{c},{t:.1f},{100 * t / tot:.1f},{t / c:.1f}\n")
    print(open(out_csv).read())


STALLS = ["wait", "short_scoreboard", "long_scoreboard", "barrier", "mio_throttle", "math_pipe_throttle",
          "not_selected", "selected", "no_instruction", "lg_throttle", "branch_resolving", "dispatch_stall",
          "drain", "membar", "sleeping", "tex_throttle", "imc_miss", "misc"]


def stalls(rep, out_txt, label):
    """Top-8 warp stall reasons per issued instruction for every kernel of a capture."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    seen = {}
    with open(out_txt, "w") as fh:
        fh.write(f"# warp stall breakdown per issued instruction (smsp__average_warps_issue_stalled_*_per_issue_active.ratio)\n")
        fh.write(f"# {label}: {rep.split('/')[-1]}; top 8 reasons per kernel\n")
        for r in data:
            name = pass_name(r[ix["Kernel Name"]], seen)
            kern = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("fdg::", "")
            us = f(r[ix["gpu__time_duration.sum"]]) if "gpu__time_duration.sum" in ix else float("nan")
            vals = []
            for st in STALLS:
                m = f"smsp__average_warps_issue_stalled_{st}_per_issue_active.ratio"
                if m in ix:
                    vals.append((f(r[ix[m]]), st))
            vals.sort(reverse=True)
            fh.write(f"{name:22s} {kern[:40]:40s} time={us:10.1f} " + " ".join(f"{st}={v:.2f}" for v, st in vals[:8]) + "\n")
    print(open(out_txt).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:7])
    elif sys.argv[1] == "stalls":
        stalls(*sys.argv[2:5])
    else:
        launches(*sys.argv[2:5])
