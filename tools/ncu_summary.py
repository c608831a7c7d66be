#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [title] > profiles/rNN_x.md
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM limit (smem)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe inst % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "FP64 tensor (DMMA) pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA inst % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# {title}\n")
    print(f"source: `{rep}` (ncu --set full --clock-control none)\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## {d.get('Kernel Name', '?')}\n")
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d and d[k] not in ("", None):
                print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(d[h]) for h in hdr
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
                  and d[h] not in ("", "0")}
        tot = sum(stalls.values()) or 1.0
        print("\nwarp-state samples (top 8):\n")
        print("| state | share |\n|---|---|")
        for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]:
            print(f"| {k} | {100 * v / tot:.1f}% |")
        print()


if __name__ == "__main__":
    main()
