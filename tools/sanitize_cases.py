"""Small invocations of every hand-written kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck) runs:

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

tcgen05/TMEM/TMA kernels included: the tensor-core VQ assignment
(k_vq_assign_tc, encode), the fused input projection + block mean
(k_input_block_mean_fwd) and the edge-tiled dW0 (k_block_mean_wgrad) in a
SAGE step with hidden 128, the TMA gather4 SQ aggregation (k_sq_mean_bulk),
the VQ fused aggregation (k_vq_mean8_fast), the sampler, GCN weights, the
bitpack kernels.  Not a test of results (the pytest suite is); sizes are
tiny so the instrumented run finishes in minutes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_14696_b200 import bitpack  # noqa: E402
from paper_2207_14696_b200.sage import SageTrainer, TrainConfig  # noqa: E402
from paper_2207_14696_b200.synth import build_sq_codec, build_vq_codec, generate_graph  # noqa: E402


def main():
    torch.cuda.set_device(0)
    n, C = 6000, 5
    dg, labels = generate_graph(n, 12.0, C, seed=0)
    train = np.arange(0, n, 5)
    for kind in ("sq4", "vq", "gcn"):
        if kind == "vq":
            dc, _ = build_vq_codec(n, 100, 4, 256, labels=labels, num_classes=C, seed=0,
                                   max_iters=3, restarts=1)
        else:
            dc = build_sq_codec(n, 128, 4 if kind == "sq4" else 8, labels=labels, num_classes=C,
                                seed=0)
        cfg = TrainConfig(fanouts=(15, 10, 5), batch_size=128, hidden=128, use_graph=False,
                          aggregator="gcn" if kind == "gcn" else "mean")
        t = SageTrainer(dg, dc, labels, C, cfg)
        t.begin_epoch(train, 0)
        for b in range(2):
            t.step(b)
        torch.cuda.synchronize()
        t.sampler.check_errors()
        print(kind, "loss", float(t.loss_buf.item()), flush=True)
    codes = np.arange(1000) % 32
    s = bitpack.pack_codes(codes, 5)
    assert np.array_equal(bitpack.unpack_codes(s, 5, 1000), codes)
    bitpack.gather_bit_rows(s, 50, np.array([0, 3, 99, 3]))
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
