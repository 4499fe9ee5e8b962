"""Write the per-round profile summaries under profiles/ from a gpurun_out capture.

usage: python scripts/summarize_profiles.py TAG ROUND_LABEL
  gpurun_out/launches_TAG.csv  (ncu --metrics gpu__time_duration.sum list of one step)
  gpurun_out/prof_TAG.ncu-rep   (ncu --set full of the bsgemm launches of one step)
-> profiles/ROUND_LABEL_launches.csv, _launches_summary.md, _gemm_ncu_full.md, traffic.json
Per-launch ncu times are cold-cache and serialised: compare shares, not absolutes.
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {  # bsgemm template -> step name (launch order within one layer step)
    "bsgemm_kernel<5, 0, 1, 64": "router", "bsgemm_kernel<0, 0, 1, 256, 0": "sdd", "bsgemm2_kernel<0, 0, 1": "sdd",
    "bsgemm_kernel<1, 0, 1, 256": "dsd+scatter", "bsgemm_kernel<0, 0, 0, 256, 1": "sddT", "bsgemm2_kernel<0, 0, 0, 1": "sddT",
    "bsgemm2_kernel<2, 1, 1": "dsTd", "bsgemm2_kernel<3, 1, 1": "ddTs",
    "bsgemm_kernel<5, 1, 1, 64": "router_dwr", "bsgemm_kernel<5, 0, 0, 128": "router_dx",
    "bsgemm_kernel<1, 0, 0, 256": "dsdT+dx",
}


OTHER = {"topo_hist": "topology", "topo_scan_emit": "topology", "scatter_rows_kernel": "gather",
         "combine_kernel": "scatter", "scatter_bwd_kernel": "scatter_bwd", "router_dwr_reduce": "router_dwr"}


def step_name(kernel):
    for k, v in OTHER.items():
        if k in kernel:
            return v
    for k, v in NAMES.items():
        if k in kernel.replace("(int)", "").replace("(bool)", ""):
            return v
    return ""


def launches(tag, label):
    src = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    rows = [r for r in rows if "moe::" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum"]
    # the last complete step: the library kernels after the last router launch
    starts = [i for i, r in enumerate(rows) if "bsgemm_kernel<(int)5, (bool)0, (bool)1, (int)64" in r["Kernel Name"]
              or "bsgemm_kernel<5, 0, 1, 64" in r["Kernel Name"]]
    if len(starts) > 1:  # a complete step: from the second-to-last router launch to the last
        step = rows[starts[-2]:starts[-1]]
        starts = []
    else:
        step = None
    if step is None:
        step = rows[starts[-1]:] if starts else rows
    shutil.copy(src, os.path.join(ROOT, "profiles", f"{label}_launches.csv"))
    tot = sum(float(r["Metric Value"]) for r in step)
    out = [f"# {label} — ncu launch list of one C1 step (gpu__time_duration.sum, --clock-control none)", "",
           f"Source: `gpurun_out/launches_{tag}.csv` (copied to `profiles/{label}_launches.csv`). "
           "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
           "| # | kernel | step | us | share of step |", "|---|---|---|---|---|"]
    for i, r in enumerate(step):
        us = float(r["Metric Value"]) / 1e3
        k = r["Kernel Name"].replace("moe::", "")
        k = re.sub(r"\(CUtensorMap_st.*", "", k)[:70]
        out.append(f"| {i} | `{k}` | {step_name(r['Kernel Name'])} | {us:.1f} | {100 * float(r['Metric Value']) / tot:.1f}% |")
    out.append(f"| | total (library kernels) | | {tot / 1e3:.1f} | 100% |")
    open(os.path.join(ROOT, "profiles", f"{label}_launches_summary.md"), "w").write("\n".join(out) + "\n")


def gemm_full(tag, label):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def g(d, k, scale=1.0):
        try:
            return float(d[ix[k]]) * scale
        except (KeyError, ValueError):
            return float("nan")
    out = [f"# {label} — ncu --set full, one C1 (MoE-XS) step, tcgen05 GEMM kernels", "",
           f"Source: `gpurun_out/prof_{tag}.ncu-rep` (ncu --set full --clock-control none --import-source on "
           "-k regex:bsgemm). Per-launch times are cold-cache, serialised, under ncu: compare shares, not absolutes.",
           "", "| step | kernel | ncu us | DRAM read MB | DRAM write MB | DRAM % peak | tensor pipe % | L2 % | issue % | regs |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    import datetime
    traffic = {"source": f"profiles/{label}_gemm_ncu_full.md (ncu --set full, dram__bytes_read.sum + "
                         f"dram__bytes_write.sum per launch, bytes; captured {datetime.date.today().isoformat()})"}
    for d in data:
        k = d[ix["Kernel Name"]]
        nm = step_name(k)
        rd, wr = g(d, "dram__bytes_read.sum"), g(d, "dram__bytes_write.sum")
        out.append(f"| {nm} | `{re.sub(r'[(]CUtensorMap.*', '', k)[:44]}` | {g(d, 'gpu__time_duration.sum'):.1f} | "
                   f"{rd:.1f} | {wr:.1f} | {g(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{g(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{g(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{g(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f} | "
                   f"{g(d, 'launch__registers_per_thread'):.0f} |")
        if nm:
            traffic[nm] = int((rd + wr) * 1e6)   # ncu reports MB here
    open(os.path.join(ROOT, "profiles", f"{label}_gemm_ncu_full.md"), "w").write("\n".join(out) + "\n")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)


def perm_full(tag, label):
    """ncu --set full of the HBM-bound non-GEMM kernels (topology, permutations,
    scatter backward): achieved DRAM GB/s against the measured copy bandwidth."""
    rep = os.path.join(ROOT, "gpurun_out", f"prof_perm_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw = float(peaks["hbm_gbs"])

    def g(d, k):
        try:
            return float(d[ix[k]])
        except (KeyError, ValueError):
            return float("nan")
    out = [f"# {label} — ncu --set full, one C1 (MoE-XS) step, non-GEMM kernels", "",
           f"Source: `gpurun_out/prof_perm_{tag}.ncu-rep` (ncu --set full --clock-control none, kernels topo_*, "
           "scatter_rows (padded gather), scatter_bwd (+ router dlogits)). DRAM GB/s = (read + write bytes) / ncu "
           f"duration, against the measured {bw:.0f} GB/s copy (MEASURED_PEAKS.json). Cold-cache, serialised.", "",
           "| kernel | ncu us | DRAM read MB | DRAM write MB | DRAM GB/s | frac of copy BW | DRAM % peak (ncu) | issue % |",
           "|---|---|---|---|---|---|---|---|"]
    seen = set()
    for d in data:
        k = re.sub(r"[(].*", "", d[ix["Kernel Name"]]).replace("moe::", "")
        if k in seen:
            continue
        seen.add(k)
        us = g(d, "gpu__time_duration.sum")
        rd, wr = g(d, "dram__bytes_read.sum"), g(d, "dram__bytes_write.sum")
        gbs = (rd + wr) * 1e6 / (us * 1e-6) / 1e9 if us > 0 else float("nan")
        out.append(f"| `{k[:48]}` | {us:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | {gbs / bw:.2f} | "
                   f"{g(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{g(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f} |")
    open(os.path.join(ROOT, "profiles", f"{label}_permute_ncu_full.md"), "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    tag, label = sys.argv[1], sys.argv[2]
    if len(sys.argv) > 3 and sys.argv[3] == "perm":
        perm_full(tag, label)
    else:
        launches(tag, label)
        gemm_full(tag, label)
