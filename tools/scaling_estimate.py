"""Per-rank cost of the cfg5 element-row partition on ONE GPU (scaling estimate).

The round's GPU budget gives one B200, so the 2/4/8-GPU strong-scaling run of
BASELINE configs[4] cannot be measured here.  This tool measures what one rank
of an N-GPU run executes: the 1024 x (1024/N) element-row block of cfg5 (same
element size, same physics and schedule) as a 1-rank NCCL partition, i.e. the
rank's kernels plus its NCCL halo send/recv and CG allreduce calls (to itself).
Estimated efficiency(N) = T_1 / (N * T_rank(N)), T_1 the single-domain cfg5
step.  Not included: NVLink transfer time of the halo (2 x 2 MiB per exchange,
~5 us at NVLink 5 rates) and the allreduce latency across GPUs (~10-20 us per
CG iteration), i.e. an upper bound on the efficiency.

A second estimate ("in_process") runs the real cfg5 problem as N in-process partitions on the one GPU:
identical CG iteration counts to an N-rank run, every kernel at its N-rank size; T_1 / T_N bounds the
efficiency from the compute side.

  python tools/scaling_estimate.py > gpurun_out/scaling_estimate.json
"""
import dataclasses
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)

import bench  # noqa: E402


def main():
    import torch
    from paper_2504_18526_b200.configs import CFG5
    from paper_2504_18526_b200.runtime import get_runtime
    torch.cuda.set_device(0)
    rt = get_runtime(0)
    rt.set_cg(rtol=1e-14, maxit=1000)
    args = bench.parse()
    out = {"workload": CFG5.name, "ranks": {}}
    r1 = bench.measure(CFG5, args, torch, rt, 0, 1, 0, 3, 3)
    t1 = r1["ms_per_step"]
    out["single_domain_ms_per_step"] = t1
    out["single_domain_cg_mean_iterations"] = r1.get("stats", r1["config"]).get("cg_mean_iterations")
    torch.cuda.empty_cache()
    for N in (2, 4, 8):
        w = dataclasses.replace(CFG5, ney=CFG5.ney // N, length_y=2 * math.pi / N)
        r = bench.measure_part(w, args, torch, rt, 0, 1, 0, 3, 3, emulate=-1)
        torch.cuda.empty_cache()
        tr = r["ms_per_step"]
        out["ranks"][N] = {"rows_per_rank": w.ney, "rank_ms_per_step": tr,
                           "rank_cg_mean_iterations": r.get("stats", r["config"]).get("cg_mean_iterations"),
                           "rank_cg_solve_us": r["roofline"]["kernel_us"],
                           "rank_cg_hbm_frac": r["roofline"]["frac"],
                           "estimated_efficiency": t1 / (N * tr),
                           "estimated_dof_sweeps_per_s": CFG5.dof_sweeps_per_step()[0] / (tr * 1e-3)}
        print(json.dumps({N: out["ranks"][N]}), file=sys.stderr, flush=True)
    # second estimate: the REAL cfg5 problem cut into N element-row partitions that one process drives on
    # this GPU one after the other (device-copy halo, fixed-order reduction): the CG iteration sequence is
    # the N-rank run's, every kernel has its N-rank size, and the step time T_N is the sum over the N
    # ranks' work, so T_N / N is a rank's compute time and T_1 / T_N the efficiency bound (again without
    # NVLink / allreduce latency, and without the overlap the ranks' second stream buys)
    out["in_process"] = {}
    for N in (2, 4, 8):
        r = bench.measure_part(CFG5, args, torch, rt, 0, 1, 0, 2, 1, emulate=N)
        torch.cuda.empty_cache()
        tn = r["ms_per_step"]
        out["in_process"][N] = {"all_partitions_ms_per_step": tn, "per_rank_ms_per_step": tn / N,
                                "cg_mean_iterations": r["stats"]["cg_mean_iterations"] if "stats" in r else None,
                                "estimated_efficiency": t1 / tn}
        print(json.dumps({"in_process": {N: out["in_process"][N]}}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.argv = sys.argv[:1]
    main()
