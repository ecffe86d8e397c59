"""Time encode_vq's assignment kernel: tensor-core screen + fp64 recheck
(fg_vq_assign) against the float64 CUDA-core path (fg_vq_assign_fp64) on a
MAG240M-shape part layout (d=768, width 8, 256 entries, cosine), and check
the codes are identical.  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2207_14696_b200 as fg  # noqa: E402
from paper_2207_14696_b200 import _native as N  # noqa: E402
from paper_2207_14696_b200.vq import METRICS, DeviceVqCodec  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    d, w, L = 768, 8, 256
    out = {}
    for metric in ("cosine", "euclidean"):
        r = np.random.default_rng(0)
        books = [r.standard_normal((L, w)).astype(np.float32) for _ in range(d // w)]
        x = torch.randn(n, d, device="cuda")
        dc = DeviceVqCodec.empty(fg.VqParams(w, L, metric=metric), d, books, n, "cuda")
        res = {}
        for name in ("fg_vq_assign", "fg_vq_assign_fp64"):
            codes = torch.empty((n, dc.num_parts), dtype=torch.int32, device="cuda")

            def run():
                N.call(name, N.ptr(x), 0, n, d, w, L, dc.num_parts, N.ptr(dc.table),
                       N.ptr(dc.entries), METRICS.index(metric), dc.bits, N.ptr(dc.rows),
                       dc.row_stride, N.ptr(codes), N.stream_handle())
            run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(3):
                run()
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / 3
            res[name] = (ms, codes.clone())
        same = torch.equal(res["fg_vq_assign"][1], res["fg_vq_assign_fp64"][1])
        flops = 2.0 * n * d * L
        out[metric] = {"rows": n, "tc_ms": round(res["fg_vq_assign"][0], 3),
                       "fp64_ms": round(res["fg_vq_assign_fp64"][0], 3),
                       "speedup": round(res["fg_vq_assign_fp64"][0] / res["fg_vq_assign"][0], 2),
                       "tc_Mrows_s": round(n / res["fg_vq_assign"][0] / 1e3, 1),
                       "distance_TFLOPs_tc": round(flops / res["fg_vq_assign"][0] / 1e9, 2),
                       "codes_identical": bool(same)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
