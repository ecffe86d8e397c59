"""Random-row gather ceiling on this GPU: how fast can a kernel pull rows of R
bytes at uniformly random indices out of a table of T bytes in HBM?  This is
the practical roofline for fg_gather_dequant_mean, whose row reads are exactly
such random gathers, next to the sequential copy peak in
MEASURED_PEAKS.json.

The probe kernel (JIT-built here; a measuring tool, not part of the library):
16-byte lanes, R/16 lanes per row, each thread keeps UNROLL independent row
loads in flight, rows are summed so nothing is dead-code eliminated.  Tables
are larger than L2; fresh random indices per launch; CUDA events around a run
of back-to-back launches."""
import json
import sys

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
#include <cuda_runtime.h>
template <int LPR, int UNROLL>
__global__ void __launch_bounds__(256) k_probe(const int4* __restrict__ x, const int64_t* __restrict__ idx,
                                               int64_t m, int4* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = (int)(t % LPR);
  const int64_t g = t / LPR;                       // row group
  const int64_t groups = (int64_t)gridDim.x * blockDim.x / LPR;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int64_t r0 = g * UNROLL; r0 < m; r0 += groups * UNROLL) {
    int4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t r = r0 + u;
      v[u] = r < m ? __ldcs(x + idx[r] * LPR + lane) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) { acc.x += v[u].x; acc.y ^= v[u].y; acc.z += v[u].z; acc.w ^= v[u].w; }
  }
  out[t] = acc;
}
void probe(torch::Tensor x, torch::Tensor idx, torch::Tensor out, int64_t row_bytes, int64_t ctas_per_sm) {
  const int64_t m = idx.numel();
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * (int)ctas_per_sm;
  auto st = at::cuda::getCurrentCUDAStream();
  const int4* xp = (const int4*)x.data_ptr();
  int4* op = (int4*)out.data_ptr();
  const int64_t* ip = idx.data_ptr<int64_t>();
  switch (row_bytes) {
    case 32: k_probe<2, 8><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 64: k_probe<4, 8><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 1064: k_probe<4, 1><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 2064: k_probe<4, 2><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 4064: k_probe<4, 4><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 16064: k_probe<4, 16><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 32064: k_probe<4, 32><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 128: k_probe<8, 8><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 256: k_probe<16, 8><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
    case 512: k_probe<32, 8><<<grid, 256, 0, st>>>(xp, ip, m, op); break;
  }
}
"""


def main():
    mod = load_inline("fg_gather_probe", cpp_sources="void probe(torch::Tensor x, torch::Tensor idx, torch::Tensor out, int64_t row_bytes, int64_t ctas_per_sm);",
                      cuda_sources="#include <ATen/cuda/CUDAContext.h>\n" + SRC, functions=["probe"],
                      extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                      verbose=False)
    dev = torch.device("cuda", 0)
    out_tab = {}
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.empty(sms * 8 * 256 * 16 * 2, dtype=torch.uint8, device=dev)
    for table_gb in (1, 7):
        for row in (32, 64, 128, 256, 512):
            n = (table_gb << 30) // row
            x = torch.ones(n * row, dtype=torch.uint8, device=dev)
            m = (64 << 20) // row  # 64 MB of rows per launch
            idxs = [torch.randint(0, n, (m,), device=dev) for _ in range(10)]
            for i in range(3):
                mod.probe(x, idxs[i], sink, row, 8)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for i in range(10):
                mod.probe(x, idxs[i], sink, row, 8)
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / 10
            rd = m * row / (ms * 1e-3) / 1e9
            tot = m * (row + 8) / (ms * 1e-3) / 1e9
            out_tab[f"{table_gb}GB_row{row}"] = {"us": round(ms * 1e3, 2), "GBps_rows": round(rd, 1),
                                                 "GBps_rows_and_idx": round(tot, 1)}
            print(table_gb, row, out_tab[f"{table_gb}GB_row{row}"], flush=True)
            del x, idxs
            torch.cuda.empty_cache()
    # in-flight sweep for 64-byte rows, 7 GB table: UNROLL x CTAs/SM
    n = (7 << 30) // 64
    x = torch.ones(n * 64, dtype=torch.uint8, device=dev)
    m = (64 << 20) // 64
    idxs = [torch.randint(0, n, (m,), device=dev) for _ in range(10)]
    for unroll, code in ((1, 1064), (2, 2064), (4, 4064), (8, 64), (16, 16064), (32, 32064)):
        for cps in (1, 2, 4, 8):
            for i in range(2):
                mod.probe(x, idxs[i], sink, code, cps)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for i in range(10):
                mod.probe(x, idxs[i], sink, code, cps)
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / 10
            inflight_kb = cps * 256 / 4 * unroll * 64 / 1024   # rows in flight per SM x 64 B
            rd = m * 64 / (ms * 1e-3) / 1e9
            key = f"sweep64_unroll{unroll}_ctas{cps}"
            out_tab[key] = {"inflight_KB_per_SM": inflight_kb, "GBps_rows": round(rd, 1),
                            "littles_law_latency_us": round(inflight_kb * 1024 * 148 / (rd * 1e9) * 1e6, 2)}
            print(key, out_tab[key], flush=True)
    if len(sys.argv) > 1:
        json.dump(out_tab, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
