"""Summarise ncu --set full captures (.ncu-rep) into the numbers kept under
profiles/: duration, launch shape, DRAM and L2 traffic with achieved GB/s,
tensor-pipe / issue / warp activity, and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/r02a_*.ncu-rep > profiles/r02_ncu_summary.json

Units come from ncu's own unit row and are normalised to bytes / us / %.
"""
import csv
import io
import json
import subprocess
import sys

_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3,
          "%": 1, "": 1}

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
    "smem_bytes": "launch__shared_mem_per_block",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_read_sectors_from_l1": "lts__t_sectors_srcunit_tex_op_read.sum",
    "l2_bytes": "lts__t_bytes.sum",
    "l1_bytes": "l1tex__t_bytes.sum",
    "tensor_pipe_active_pct_elapsed": "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_active_pct_alt": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct_elapsed": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "tensor_mem_active_pct_of_active_sm": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_pipe_inst_pct_of_active_sm": "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "tc_pipe_inst_pct_max_sm": "sm__inst_executed_pipe_tc.max.pct_of_peak_sustained_active",
    "hmma_subpipe_inst_pct_of_active_sm": "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram_pct_peak": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def num(x, unit):
    try:
        return float(x.replace(",", "")) * _SCALE.get(unit, 1)
    except ValueError:
        return None


def summarise(rep):
    head, units, rows = raw(rep)
    res = []
    for row in rows:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        s = {"kernel": d.get("Kernel Name", "?"), "rep": rep}
        for k, m in KEYS.items():
            if m in d:
                s[k] = num(d[m], u.get(m, ""))
        if s.get("tensor_pipe_active_pct_elapsed") is None and s.get("tensor_pipe_active_pct_alt") is not None:
            s["tensor_pipe_active_pct_elapsed"] = s["tensor_pipe_active_pct_alt"]
        s.pop("tensor_pipe_active_pct_alt", None)
        if s.get("l2_read_sectors_from_l1") is not None:
            s["l2_read_bytes_from_l1"] = 32 * s["l2_read_sectors_from_l1"]
        t = s.get("duration_us")
        if t:
            dram = (s.get("dram_read_bytes") or 0) + (s.get("dram_write_bytes") or 0)
            s["dram_bytes"] = dram
            s["dram_GBps"] = dram / t / 1e3
            if s.get("l2_bytes"):
                s["l2_GBps"] = s["l2_bytes"] / t / 1e3
            if s.get("l2_read_bytes_from_l1"):
                s["l2_read_from_l1_GBps"] = s["l2_read_bytes_from_l1"] / t / 1e3
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
                x = num(v, "")
                if x:
                    stalls[k[len("smsp__average_warp_latency_issue_stalled_"):-len(".ratio")]] = x
        if stalls:
            s["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        res.append(s)
    return res


if __name__ == "__main__":
    out = []
    for rep in sys.argv[1:]:
        out.extend(summarise(rep))
    json.dump(out, sys.stdout, indent=1)
    sys.stdout.write("\n")
