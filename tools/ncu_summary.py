#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into markdown for profiles/.

    python tools/ncu_summary.py report.ncu-rep [--title T] > profiles/rNN_kernel.md
    python tools/ncu_summary.py launches.csv --launches > profiles/rNN_launches.md
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum", "UTCHMMA fp16->fp32 ops"),
    ("sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
     "UTCHMMA % of peak (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__sass_inst_executed_op_utcmma.sum", "UTCMMA instructions"),
    ("smsp__sass_inst_executed_op_tmem_ldt.sum", "tcgen05.ld instructions"),
    ("smsp__sass_inst_executed_op_tmem_stt.sum", "tcgen05.st instructions"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def raw_rows(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(r, dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def summarise_report(rep: str, title: str | None) -> str:
    lines = []
    for _, vals, units in raw_rows(rep):
        name = vals.get("Kernel Name", "?")
        lines.append(f"## {title or name}\n")
        lines.append(f"`{name}`  (source: `{rep}`, `ncu --set full --clock-control none`)\n")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for key, label in METRICS:
            if key in vals:
                lines.append(f"| {label} (`{key}`) | {vals[key]} | {units.get(key, '')} |")
        stalls = [(k[len(STALLS):].replace("_per_issue_active.ratio", ""), float(v))
                  for k, v in vals.items()
                  if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio") and v]
        stalls = sorted(stalls, key=lambda kv: -kv[1])[:8]
        if stalls:
            lines.append("\nTop warp stall reasons (cycles per issued instruction):\n")
            lines.append("| reason | cycles |")
            lines.append("|---|---|")
            for k, v in stalls:
                lines.append(f"| {k} | {v:.2f} |")
        lines.append("")
    return "\n".join(lines)


def summarise_launches(path: str) -> str:
    """Per-kernel launch count, time and share; DRAM bytes per launch when the list
    also carries dram__bytes_read/write.sum (several metrics per launch)."""
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    im = hdr.index("Metric Name") if "Metric Name" in hdr else None
    tot = collections.defaultdict(float)
    dram = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = ""
    scales = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
              "msecond": 1.0}
    bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[1:]:
        if len(r) <= iv or not r[iv]:
            continue
        v = float(r[iv].replace(",", ""))
        name = r[ik].split("(")[0]
        metric = r[im] if im is not None else "gpu__time_duration.sum"
        if metric.startswith("dram__bytes"):
            dram[name] += v * bscale.get(r[iu], 1.0)
            continue
        if metric != "gpu__time_duration.sum":
            continue
        tot[name] += v * scales.get(r[iu], 1.0)
        cnt[name] += 1
    grand = sum(tot.values())
    has_dram = bool(dram)
    lines = [f"Launch list `{path}` (`ncu --metrics gpu__time_duration.sum"
             f"{',dram__bytes_read.sum,dram__bytes_write.sum' if has_dram else ''}"
             " --clock-control none`, serialised, cold cache)\n",
             "| kernel | launches | total ms | mean ms | share |" +
             (" DRAM GB / launch |" if has_dram else ""),
             "|---|---|---|---|---|" + ("---|" if has_dram else "")]
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        row = f"| `{name}` | {cnt[name]} | {t:.3f} | {t / cnt[name]:.3f} | {t / grand:.1%} |"
        if has_dram:
            row += f" {dram[name] / cnt[name] / 1e9:.2f} |"
        lines.append(row)
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--title")
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args()
    sys.stdout.write(summarise_launches(a.path) if a.launches else summarise_report(a.path, a.title))


if __name__ == "__main__":
    main()
