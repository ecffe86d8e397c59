"""CPU cost of the reference's fit_vq inner loop (oracle restatement of
vq.py:166-254, float64 numpy/OpenBLAS): one part, one restart, on a
sample of `rows` rows -- the unit the full fit repeats parts x restarts
times.  Used to put the GPU fit time (bench's "[synth] vq codec: fit_vq ..."
line) next to the reference's.  Runs on the CPU only; not a bench line."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import codecs as oc  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    width = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    length = int(sys.argv[3]) if len(sys.argv) > 3 else 256
    rng = np.random.default_rng(0)
    s = rng.standard_normal(width)
    pts = np.sqrt(0.9) * s + np.sqrt(0.1) * rng.standard_normal((rows, width))
    pts /= np.linalg.norm(pts, axis=1, keepdims=True)          # cosine parts are normalised
    t0 = time.perf_counter()
    _, obj, hist = oc.lloyd(pts, length, "cosine", 50, 1e-4, np.random.default_rng(1))
    dt = time.perf_counter() - t0
    print(f"rows {rows} width {width} L {length}: one part x one restart "
          f"{dt:.2f} s ({len(hist) - 1} Lloyd iterations), threads "
          f"{os.environ.get('OPENBLAS_NUM_THREADS', 'default')}, cores {os.cpu_count()}")


if __name__ == "__main__":
    main()
