"""Summarise a round's ncu launch list + full capture into profiles/.

python tools/summarize_profile.py r01 [config]
writes profiles/<tag>_launches.csv (copy), profiles/<tag>_ncu_summary.md and
profiles/deep_traffic.json (DRAM bytes per deep launch, read by bench.py).
"""
import csv
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
config = sys.argv[2] if len(sys.argv) > 2 else "c4"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)

# launch list: per-kernel mean duration and share
rows = [r for r in csv.reader(open(os.path.join(go, f"{tag}_launches.csv"))) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
iu = hdr.index("Metric Unit")
to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
per = {}
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr) or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("void ", "").strip()
    per.setdefault(name, []).append(float(r[iv].replace(",", "")) * to_us.get(r[iu], 1.0))
shutil.copy(os.path.join(go, f"{tag}_launches.csv"), os.path.join(prof, f"{tag}_launches.csv"))

raw = subprocess.run(["ncu", "-i", os.path.join(go, f"{tag}_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout.splitlines()
R = list(csv.reader(raw))
H, U = R[0], R[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg"]
caps = []
OPS = ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"]
for r in R[2:]:
    d = {"kernel": r[H.index("Kernel Name")].split("(")[0].replace("void ", "").strip()}
    for w in want:
        if w in H:
            d[w] = r[H.index(w)] + (" " + U[H.index(w)] if U[H.index(w)] else "")
    # ncu-measured FP64 work (SURVEY 8d cross-check): 2 DFMA + DADD + DMUL
    # thread-ops, from the per-cycle rates times the elapsed cycles
    if all(o in H for o in OPS) and "sm__cycles_elapsed.avg" in H:
        cyc = float(r[H.index("sm__cycles_elapsed.avg")].replace(",", ""))
        fma, dadd, dmul = (float(r[H.index(o)].replace(",", "")) * cyc for o in OPS)
        d["fp64 flops (2 dfma + dadd + dmul, ncu)"] = f"{2 * fma + dadd + dmul:.4g}"
    caps.append(d)
want.append("fp64 flops (2 dfma + dadd + dmul, ncu)")

lines = [f"# {tag} ncu summary (config {config}, bench.py --steps 3 --warmup 3)", "",
         "## Launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)", "",
         "| kernel | launches | mean us | share |", "|---|---|---|---|"]
tot = sum(sum(v) for v in per.values())
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}% |")
lines += ["", "(`dfma_probe_kernel` is bench.py's live FP64-peak measurement, outside the timed steps.)"]
lines += ["", "## --set full captures", ""]
for d in caps:
    lines.append(f"### `{d['kernel']}`")
    for w in want:
        if w in d:
            lines.append(f"- {w}: {d[w]}")
    lines.append("")
open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")

deep = [d for d in caps if "deep_kernel" in d["kernel"] or "deep_tpc_kernel" in d["kernel"]]
if deep:
    d = deep[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(k):
        f = d[k].split()
        return float(f[0]) * scale.get(f[1] if len(f) > 1 else "byte", 1)
    # the library's own name for the launch (cvg_last_deep_kernel), from the
    # template arguments <VAR, warps, regcap, lanes per column, k-order, fused>
    # and the grid (blocks per SM over 148 SMs)
    desc = None
    m = __import__("re").search(r"deep_tpc_kernel<(\d+), (\d+), (\d+), (\d+), (\d+)", d["kernel"])
    if m:
        grid = int(float(d.get("launch__grid_size", "148").split()[0]))
        desc = (f"deep_tpc_kernel<lanes_per_column={m.group(4)},k_order_precip={m.group(5)},warps={m.group(2)},"
                f"blocks_per_sm={max(1, grid // 148)}>")
    # DRAM bytes of one default step: the first capture of each kernel of the
    # default schedule (trigger, deep, re-derivation, shallow)
    def dram(x):
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            f = x[k].split()
            tot += float(f[0]) * scale.get(f[1] if len(f) > 1 else "byte", 1)
        return tot
    step, seen = {}, set()
    for x in caps:
        base = x["kernel"].split("<")[0]
        if base in seen:
            continue
        seen.add(base)
        step[x["kernel"]] = dram(x)
    prev = {}
    try:   # keep the range capture of the overlapped step (tools/step_range.py), if any
        prev = json.load(open(os.path.join(prof, "deep_traffic.json")))
    except Exception:
        pass
    keep = {k: prev[k] for k in ("step_dram_bytes_overlapped", "step_range_source") if k in prev}
    json.dump({**keep, "config": config, "tag": tag, "kernel": d["kernel"], "kernel_desc": desc,
               "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
               "step_dram_bytes": sum(step.values()), "step_dram_bytes_by_kernel": step,
               "source": f"profiles/{tag}_ncu_summary.md (ncu --set full, one launch of each kernel, serialised)"},
              open(os.path.join(prof, "deep_traffic.json"), "w"), indent=1)
print("\n".join(lines))
