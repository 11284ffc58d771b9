# SPDX-License-Identifier: Apache-2.0
"""Summarise an ncu --set full report (tools/profile_round.sh) into the JSON kept under
profiles/: per kernel duration, DRAM bytes, tensor-pipe activity and bf16 UTC MMA
throughput vs peak, SM / DRAM throughput, clock, registers.
usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/ncu_<round>_kernels.json"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name, scale=1.0):
    if name not in col or not r[col[name]]:
        return None
    x = float(r[col[name]].replace(",", ""))
    u = units[col[name]]
    mult = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,  # -> ms
            "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0,        # -> GB
            "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}.get(u, 1.0)    # -> GHz
    return round(x * mult * scale, 6)


out = []
for r in rows[2:]:
    out.append({
        "kernel": r[col["Kernel Name"]],
        "duration_ms": val(r, "gpu__time_duration.sum"),
        "dram_read_GB": val(r, "dram__bytes_read.sum"),
        "dram_write_GB": val(r, "dram__bytes_write.sum"),
        "tensor_pipe_active_pct": val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "bf16_mma_pct_of_peak": val(r, "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"),
        # SMEM data pipe: tensor-core operand reads + thread (LSU) shared loads / stores
        "smem_tc_wavefronts_pct": val(r, "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_lsu_wavefronts_pct": val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "smem_bank_reads_pct": val(r, "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed"),
        "smem_bank_writes_pct": val(r, "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed"),
        "sm_throughput_pct": val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_clock_GHz": val(r, "sm__cycles_elapsed.avg.per_second"),
        "regs": val(r, "launch__registers_per_thread"),
    })
print(json.dumps({"_note": f"ncu --set full --clock-control none, one launch each ({rep}); units ms, GB, GHz",
                  "kernels": out}, indent=1))
