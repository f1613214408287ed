"""Top-K in the bench's own context (tuning helper): the DecodeModel of bench.py with 4 layers,
31 timed steps, then the bench's Top-K and dense per-launch measurements."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2303_06865_b200 import flexq as fq  # noqa: E402
from paper_2303_06865_b200 import workloads as wl  # noqa: E402


def main():
    w = wl.CONFIGS["opt-175b"]
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    m = bench.DecodeModel(w, 4, w.batch, 0, w.batch, bench.synth_seed(), dev, st, True)
    m.capture()
    m.time_steps(3, 31, torch.cuda.synchronize)
    cur = w.prompt_len + m.steps_i[-1]   # the bench's cur_last
    res = {"cur_len": cur, "keep": fq.topk_keep(cur), "lib": os.environ.get("FLEXQ_LIB", "default")}
    for rep in range(2):
        res[f"topk_tm_{rep}"] = round(m.per_launch(cur, "topk_tm", layers=4), 2)
        res[f"attn_{rep}"] = round(m.per_launch(cur, "attn", layers=4), 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
