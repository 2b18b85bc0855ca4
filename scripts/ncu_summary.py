#!/usr/bin/env python
"""Summarise an ncu --set full report: SOL, memory, occupancy, top stall reasons."""
import csv, io, subprocess, sys

KEEP = {"GPU Speed Of Light Throughput": ["Duration", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput"],
        "Memory Workload Analysis": ["L1/TEX Hit Rate", "L2 Hit Rate", "Mem Pipes Busy"],
        "Compute Workload Analysis": ["Executed Ipc Active", "Issue Slots Busy"],
        "Occupancy": ["Achieved Occupancy", "Theoretical Occupancy", "Block Limit Shared Mem",
                      "Block Limit Registers"],
        "Launch Statistics": ["Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block"],
        "Scheduler Statistics": ["Eligible Warps Per Scheduler", "No Eligible"],
        "Warp State Statistics": ["Warp Cycles Per Issued Instruction"]}


def run(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    print(f"== {rep}")
    name = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Kernel Name") != name:
            name = d.get("Kernel Name")
            print("kernel:", name[:110])
        if d.get("Metric Name") in KEEP.get(d.get("Section Name"), []):
            print(f"  {d['Metric Name']:<36} {d['Metric Value']:>14} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rr[0], rr[1], rr[2]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
            "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
            "smsp__sass_inst_executed_op_shared_atom.sum", "smsp__inst_executed_op_global_red.sum",
            "lts__t_sectors_srcunit_tex_op_red.sum",
            "lts__t_sectors_srcunit_tex_op_red.sum.pct_of_peak_sustained_elapsed",
            "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
    for k in want:
        if k in h:
            i = h.index(k)
            print(f"  {k:<58} {vals[i]:>16} {units[i]}")
    pipes = []
    for k, v in zip(h, vals):
        if k.startswith("sm__inst_executed_pipe_") and k.endswith("pct_of_peak_sustained_active"):
            try:
                pipes.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
    pipes.sort(reverse=True)
    for v, k in pipes[:6]:
        print(f"  pipe {k:<70} {v:>8.1f} %")
    stalls = [(k, v) for k, v in zip(h, vals) if k.startswith("smsp__average_warp_latency_issue_stalled_")
              or k.startswith("smsp__pcsamp_warps_issue_stalled_")]
    st = []
    for k, v in stalls:
        try:
            st.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
    st.sort(reverse=True)
    for v, k in st[:8]:
        print(f"  stall {k:<70} {v:>12.1f}")


for rep in sys.argv[1:]:
    run(rep)
