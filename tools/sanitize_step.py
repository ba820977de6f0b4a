"""Config-A training steps for compute-sanitizer (SURVEY §4 tier 7):

    compute-sanitizer --tool memcheck  python tools/sanitize_step.py
    compute-sanitizer --tool racecheck python tools/sanitize_step.py

Runs the product path on config A's shape (<= 20-atom molecules, L = 2, H = 32 channel-padded
to 128, batch 64): eager forward/backward/AdamW, two graph-replayed steps and an eval batch,
then synchronises through hg_sync; prints one line. One tool per GPU call (B200_PROFILING.md)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import molgen  # noqa: E402
from paper_2207_11333_b200 import hgnn  # noqa: E402


def main():
    data = molgen.generate("tiny", 300, 1)
    store = hgnn.Store(data)
    B = 64
    nn = np.diff(data["node_offset"])
    ne = np.diff(data["edge_offset"])
    delta = store.degree_stat()
    cfg = hgnn.make_config(data["f_node"], 4, 32, 2, B, int(np.sort(nn)[-B:].sum()), int(np.sort(ne)[-B:].sum()),
                           delta, max_degree=store.stats()["max_degree"])
    ctx = hgnn.Context(cfg)
    ctx.params_init(2)
    ids = hgnn.hg_shard(3, 0, 0, 1, len(data["y"]))
    ctx.pack(store, ids[:B], 0)
    ctx.train_step(0, graph=False)
    for k in range(2):
        ctx.pack(store, ids[(k + 1) * B:(k + 2) * B], (k + 1) % 2)
        ctx.train_step((k + 1) % 2, graph=True)
    ctx.eval_reset()
    ctx.eval_batch(0)
    ctx.sync()
    print("sanitize_step ok: loss", ctx.loss(), "eval", ctx.eval_result(), "launches", ctx.launch_count())


if __name__ == "__main__":
    main()
