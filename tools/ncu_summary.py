"""Summarise an ncu --set full report (raw page CSV) per kernel: time, DRAM bytes, throughput.
Usage: ncu -i X.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv [traffic.json] [skip]
skip: leading kernels excluded from the per-timer traffic (e.g. the index build's Map + digit pass,
which run at load time before the first step)."""
import csv
import json
import sys

import gzip
opener = gzip.open if sys.argv[1].endswith(".gz") else open
rows = list(csv.reader(opener(sys.argv[1], "rt")))
h, units = rows[0], rows[1]
SKIP = int(sys.argv[3]) if len(sys.argv) > 3 else 0
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1}


def get(r, name):
    i = h.index(name)
    return r[i], units[i]


traffic = {}
runs = {}  # kernel -> number of runs of consecutive launches (one library timer invocation may
prev = None  # launch a kernel twice in a row, e.g. the expansion's full tiles + its last tile)
print("| kernel | grid | regs | time ms | DRAM read GB | DRAM write GB | DRAM GB/s | DRAM % peak | SM % | issued inst |")
print("|---|---|---|---|---|---|---|---|---|---|")
for ri, r in enumerate(rows[2:]):
    name = get(r, "Kernel Name")[0].split("(")[0].split("::")[-1]
    short = name.split("<")[0].replace("_kernel", "")
    t, tu = get(r, "gpu__time_duration.sum")
    t = float(t) * tscale[tu]
    rd, ru = get(r, "dram__bytes_read.sum")
    wr, wu = get(r, "dram__bytes_write.sum")
    rd, wr = float(rd) * scale[ru], float(wr) * scale[wu]
    dpct = get(r, "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed")[0]
    smpct = get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")[0]
    regs = get(r, "launch__registers_per_thread")[0]
    grid = get(r, "launch__grid_size")[0]
    inst = get(r, "smsp__inst_executed.sum")[0]
    print(f"| {name} | {grid} | {regs} | {t*1e3:.3f} | {rd/1e9:.3f} | {wr/1e9:.3f} | "
          f"{(rd+wr)/t/1e9:.0f} | {dpct} | {smpct} | {inst} |")
    if ri >= SKIP:
        traffic.setdefault(short, []).append(rd + wr)
        if short != prev:
            runs[short] = runs.get(short, 0) + 1
    prev = short
# DRAM bytes per invocation of each library timer (bench.py's kernel names): a timer may cover
# several kernels; its invocations are counted by its anchor kernel
TIMERS = {  # timer: (member kernels, invocations from the launch counts)
    "radix_pass": (["radix_pass"], lambda c: c("radix_pass")),
    "filter_build": (["filter_build", "filter_sample", "cfilter_build", "cfilter_sample",
                      "wfilter_build", "wfilter_sample"],
                     lambda c: c("filter_build") + c("cfilter_build") + c("wfilter_build")),
    "filter_probe": (["sj_probe_stage", "sj_probe_stage16"],
                     lambda c: c("sj_probe_stage") + c("sj_probe_stage16")),
    "filter_gather": (["sj_gather"], lambda c: c("sj_gather")),
    "filter_set": (["sj_set_words"], lambda c: c("sj_set_words")),
    "pack_hist": (["pack_hist"], lambda c: c("pack_hist")),
    "find_groups": (["find_groups"], lambda c: c("find_groups")),
    "expand": (["expand"], lambda c: c("expand", runs=True)),
    "verify_emit": (["verify_emit"], lambda c: c("verify_emit")),
    "scan_write": (["scan_write"], lambda c: c("scan_write")),
}
per_timer = {}
for timer, (members, inv_of) in TIMERS.items():
    inv = inv_of(lambda k, runs_=runs, **kw: runs_.get(k, 0) if kw.get("runs") else len(traffic.get(k, [])))
    if inv:
        per_timer[timer] = sum(sum(traffic.get(m, [])) for m in members) / inv
if len(sys.argv) > 2:
    per_timer["_note"] = ("DRAM bytes read+written per invocation of each library timer, from one "
                          "ncu --set full capture of one bench step (tools/ncu_summary.py)")
    json.dump(per_timer, open(sys.argv[2], "w"), indent=1)
