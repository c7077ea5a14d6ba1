"""The paper's Fig. 3 error sweep (maximally mixed state, mean HS distance and
infidelity vs N0) on one B200: records drawn by the device generator and
streamed through the pipeline (reconstruct_generated), metrics on the device.

    python tools/fig3_sweep.py --n 14 --n0 1 2 4 --trials 2 > profiles/r01_fig3_n14.json
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10)
    ap.add_argument("--n0", type=int, nargs="+", default=[1, 4, 16])
    ap.add_argument("--trials", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    import torch

    from paper_1602_08604_b200 import metrics

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = []
    for n0 in a.n0:
        t = time.perf_counter()
        r = metrics.error_scaling(a.n, [n0], a.trials, seed=a.seed)[0]
        r["wall_s_per_trial"] = (time.perf_counter() - t) / a.trials
        r["ratio_hs_mu_to_pred"] = r["mean_hs_mu"] / r["pred_hs"]
        r["ratio_infid_to_pred"] = r["mean_infidelity"] / r["pred_infid"]
        rows.append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps({"n": a.n, "trials": a.trials, "seed": a.seed, "shots_per_setting": "d*N0",
                      "wall_s": time.perf_counter() - t0, "rows": rows}))


if __name__ == "__main__":
    main()
