#!/usr/bin/env python3
"""Per-kernel roofline table of the tensor-core edge kernels (pair mode) on the C2
workload (one B200): each kernel timed with the step's concurrency (all 32
micro-batches launched on the 32 lanes with the step's grids, CUDA events
around whole rounds; janus_stage_time_edge_kernel mb = -1) and as an
isolated single-micro-batch launch; executed MMA FLOPs per directed edge
(pair kernels: per pair / 2; stage.cu pair_flops_per_edge); fraction of the
measured bf16 dense peak (MEASURED_PEAKS.json).  ncu metrics per kernel come
from `--set full` captures (tools/capture_profiles.sh) and are merged in by
--ncu-csv name=path pairs (raw page CSV)."""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_18404_b200 as J  # noqa: E402

# timing hook index -> what it launches (stage.cu launch_edge_kernel, pair mode)
NAMES = {0: "msg_filter_tc + msg_fe_rows", 1: "msg_ff_rows", 2: "msg_bf_pair_tc + msg_bf_rows",
         3: "msg_be_pair_tc + msg_be_rows", 4: "msg_bf_pair_tc", 5: "msg_be_pair_tc"}
NCU = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "launch__grid_size")


def ncu_metrics(path):
    rows = list(csv.reader(open(path)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[h.index(k)], u[h.index(k)]) for k in NCU if k in h}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ncu-csv", nargs="*", default=[])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "kernel_roofline.json"))
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = peaks["bf16_tflops"]
    model = J.Model(L=4, H=64, R=64, precision=J.PREC_TF32)
    params = model.synth_params(7)
    batches = [J.synth_batch(model, [256], 0.095, 700 + i, device_nl=True) for i in range(32)]
    tr = J.Trainer(model, params, 1, J.METHOD_SYMFOLD, 32, max_atoms=256, max_edges=256 * 140, max_struct=1,
                   graphs=True, lanes=32)
    tr.load_many(batches)
    for _ in range(3):
        tr.step()
    st = tr.stage(0)
    ncu = dict(x.split("=", 1) for x in args.ncu_csv)
    rows = []
    for w, name in NAMES.items():
        ms, e, fl = st.time_edge_kernel(w, -1, iters=20)
        ims, ie, ifl = st.time_edge_kernel(w, 0, iters=50)
        r = {"kernel": name, "flop_per_edge": fl / e, "step_concurrency_tflops": fl / (ms * 1e-3) / 1e12,
             "frac_of_bf16_peak": fl / (ms * 1e-3) / 1e12 / peak, "round_ms_32_microbatches": ms,
             "isolated_launch_us": ims * 1e3, "isolated_tflops": ifl / (ims * 1e-3) / 1e12}
        if name in ncu:
            r["ncu"] = ncu_metrics(ncu[name])
        rows.append(r)
        print(json.dumps(r), flush=True)
    tr.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"peak_bf16_tflops": peak, "workload": "C2: 32 x 256-atom cells, L=4 H=64, 32 lanes", "rows": rows},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
