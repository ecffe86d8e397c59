/*
 * featgrind-b200 — C ABI of the B200-native compressed-feature GNN
 * mini-batch path (arxiv 2207.14696 / reference package `featgrind`).
 *
 * Every entry point takes plain device pointers and sizes plus a
 * cudaStream_t passed as `void*`; nothing here mentions torch.  The caller
 * owns and allocates all memory (including workspaces); the library never
 * allocates or frees caller memory and keeps no global mutable state apart
 * from a thread-local error string.  All launches are stream-ordered and
 * capture-safe (no host synchronisation, no implicit allocation), so a whole
 * training step can be recorded into one CUDA graph.
 *
 * Return codes mirror the reference's error convention
 * (pkg/src/featgrind/errors.py:8-13, cli.py:46-52,503-505):
 *   FG_OK 0, FG_EUSAGE 1 (bad arguments), FG_EDATA 2 (bad data, e.g. a row
 *   id out of range -> DataError), FG_ECUDA 3 (CUDA runtime failure).
 * Device-detected data errors are reported through an `int32_t* err_flag`
 * (device memory, caller-zeroed) that the host checks when it chooses to.
 *
 * Device code-row layout ("rows"): the reference payload is one continuous
 * MSB-first bitstream, row r starting at bit r*row_bits
 * (pkg/src/featgrind/bitpack.py:17-83, sq.py:61-81).  On the device each row
 * starts on its own `row_stride`-byte boundary (stride a multiple of 16,
 * normally 32 so a row never straddles more sectors than it must); bit order
 * inside a row is unchanged.  fg_stream_to_rows / fg_rows_to_stream convert.
 */
#ifndef FEATGRIND_B200_H
#define FEATGRIND_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_OK 0
#define FG_EUSAGE 1
#define FG_EDATA 2
#define FG_ECUDA 3

/* output element types for decode / aggregate */
#define FG_OUT_F32 0
#define FG_OUT_BF16 1
#define FG_OUT_F64 2

/* aggregators (fg_block_edge_weights) */
#define FG_AGG_MEAN 0
#define FG_AGG_GCN 1

#define FG_CODEC_SQ 1
#define FG_CODEC_VQ 2

#define FG_METRIC_EUCLIDEAN 0 /* vq.py:29 METRICS order */
#define FG_METRIC_COSINE 1

/* Device-resident codec: what the gather / aggregate kernels read. */
typedef struct fg_codec_desc {
  int32_t kind;        /* FG_CODEC_SQ | FG_CODEC_VQ */
  int32_t bits;        /* SQ: k (1..8); VQ: bits per code (1..16) */
  int64_t n;           /* rows */
  int64_t d;           /* feature dim */
  int64_t row_stride;  /* bytes between device rows (multiple of 16) */
  const uint8_t* rows; /* n * row_stride bytes */
  const void* table;   /* SQ: LUT of 2^k values (float, or double for
                          elem_bits 64); VQ: float codebooks [P][L][width],
                          narrow last part zero-padded to width */
  int32_t width;       /* VQ: dims per part */
  int32_t length;      /* VQ: entries per part (padded) */
  int32_t num_parts;   /* VQ: ceil(d / width) */
  int32_t elem_bits;   /* 32 or 64: decode precision of the table */
  const void* table_lp; /* optional bf16 copy of a VQ table (same layout);
                           used only by bf16-output aggregation, may be NULL */
  const void* table_h;  /* optional fp16 copy of a VQ table, part p scaled by
                           2^s_p so its largest |entry| is <= 2048 and every
                           nonzero entry is a normal fp16 (the bf16-output
                           mean accumulates it with HADD2 in chunks of <= 8
                           picks); may be NULL (then table_lp is used) */
  const float* part_scale; /* [num_parts] 2^-s_p (device), with table_h */
} fg_codec_desc;

/* ------------------------------------------------------------ library */
const char* fg_last_error(void);
int fg_version(void);               /* 100 * major + minor */
/* Number of kernels this library has launched in the process so far
 * (benchmarks report launches per step from it). */
int64_t fg_launch_count(void);
int fg_sm_count(int* out);
/* Device-wide L2 fetch granularity for global-memory misses
 * (cudaLimitMaxL2FetchGranularity: 32 / 64 / 128 bytes; 0 = leave as is).
 * The fused gathers read small random code rows (25-96 B): a wider fetch
 * than the row wastes DRAM bandwidth.  Set once per process by the Python
 * facade from FG_L2_FETCH (default: leave the driver's setting). */
int fg_set_l2_fetch_granularity(int bytes);
int fg_get_l2_fetch_granularity(int* out);

/* -------------------------------------------------------- code layout */
/* Continuous reference stream (bitpack.py:17-36 layout, row_bits per row)
 * <-> strided device rows.  Replaces the byte-window gather of
 * bitpack.py:58-83 (gather_bit_rows) with a one-time repack on upload. */
int fg_stream_to_rows(const uint8_t* stream, int64_t stream_bytes, int64_t n,
                      int64_t row_bits, uint8_t* rows, int64_t row_stride,
                      void* cuda_stream);
int fg_rows_to_stream(const uint8_t* rows, int64_t n, int64_t row_bits,
                      int64_t row_stride, uint8_t* stream, int64_t stream_bytes,
                      void* cuda_stream);

/* The reference's bitpack module itself (Python facade
 * paper_2207_14696_b200/bitpack.py, same names and errors):
 *   fg_bits_pack        <- pack_codes(codes, bits)         bitpack.py:17-36
 *                          int64 codes -> ceil(count*bits/8) stream bytes;
 *                          a code < 0 or >= 2^bits sets *err_flag
 *                          ("codes do not fit in N bits");
 *   fg_bits_unpack      <- unpack_codes(payload, bits, count, start_bit)
 *                          bitpack.py:39-55; FG_EDATA when the stream is
 *                          shorter than start_bit + count*bits;
 *   fg_bit_rows_gather  <- gather_bit_rows(payload, row_bits, row_ids)
 *                          bitpack.py:58-83: out[nrows][row_bits] of 0/1
 *                          bytes; a row past the stream sets *err_flag
 *                          ("row ids exceed the packed stream").
 * bits in [1, 32] (else FG_EUSAGE). */
int fg_bits_pack(const int64_t* codes, int64_t count, int bits, uint8_t* out,
                 int32_t* err_flag, void* cuda_stream);
int fg_bits_unpack(const uint8_t* stream, int64_t stream_bytes, int64_t start_bit,
                   int64_t count, int bits, int64_t* out, void* cuda_stream);
int fg_bit_rows_gather(const uint8_t* stream, int64_t stream_bytes, int64_t row_bits,
                       const int64_t* rows, int64_t nrows, uint8_t* out,
                       int32_t* err_flag, void* cuda_stream);

/* ----------------------------------------------------------------- SQ */
/* quantize_sq (sq.py:114-129).  `thresholds` (device, float, 2^(k-1)-1
 * entries, ascending) are the smallest |x| whose reference code offset is
 * >= j, j = 1..2^(k-1)-1, derived on the host from the reference formula;
 * code = half + #(t_j <= |x|) for x >= 0 (including -0.0), else
 * half - 1 - #.  k = 1 ignores thresholds (code = x >= 0).  `x` is row-major
 * float32 (x_is_f64 = 0) or float64 (x_is_f64 = 1). */
int fg_sq_encode(const void* x, int x_is_f64, int64_t n, int64_t d, int k,
                 const float* thresholds, const double* thresholds64,
                 uint8_t* rows, int64_t row_stride, void* cuda_stream);

/* dequantize_sq(c, rows) (sq.py:132-153) for a device id list:
 * out[i, :] = table[code(ids[i], :)].  ids are int64 (ids_are_i32 = 0) or
 * int32.  Out-of-range ids set *err_flag = FG_EDATA and write nothing for
 * that row. */
int fg_sq_gather_dequant(const fg_codec_desc* codec, const void* ids,
                         int ids_are_i32, int64_t num_ids, void* out,
                         int out_dtype, int32_t* err_flag, void* cuda_stream);

/* fit_sq support (sq.py:96-106): count nonzeros of a float32 matrix. */
int fg_count_nonzero(const float* x, int64_t count, unsigned long long* out_count,
                     void* cuda_stream);
/* Gather |x| of the nonzeros at the evenly strided ranks the reference's
 * np.linspace(0, nnz-1, cap).astype(int64) selects (or all nonzeros when
 * nnz <= cap), preserving row-major order.  out has min(nnz, cap) floats. */
int fg_gather_nonzero_sample(const float* x, int64_t count, int64_t nnz,
                             int64_t cap, float* out_abs, void* workspace,
                             int64_t workspace_bytes, void* cuda_stream);
int64_t fg_nonzero_sample_workspace_bytes(int64_t count);
/* Streaming form: x is one row-major chunk of a larger matrix whose first
 * nonzero has global rank rank_base; nnz is the whole matrix's nonzero count
 * and out_abs the whole sample (min(nnz, cap) floats): the chunk writes the
 * picks whose global rank it holds. */
int fg_gather_nonzero_sample_chunk(const float* x, int64_t count, int64_t rank_base,
                                   int64_t nnz, int64_t cap, float* out_abs,
                                   void* workspace, int64_t workspace_bytes,
                                   void* cuda_stream);
/* k-th smallest (0-based) of non-negative floats, for each requested rank;
 * two-pass 16-bit radix select.  Exact (returns the element bit pattern).
 * Synchronises `cuda_stream` (offline fit path; not graph-capturable). */
int fg_select_ranks(const float* vals, int64_t count, const int64_t* ranks_host,
                    int num_ranks, float* out_host, void* workspace,
                    int64_t workspace_bytes, void* cuda_stream);
int64_t fg_select_workspace_bytes(void);

/* ----------------------------------------------------------------- VQ */
/* encode_vq (vq.py:306-327): per row and part, nearest codebook entry in
 * float64 arithmetic ordered as numpy/OpenBLAS evaluate the reference
 * expressions (FMA-chained dot products, numpy pairwise add.reduce for norms);
 * ties -> lowest index; cosine zero sub-vectors -> 0.  `books` is float32
 * [P][L][width] (fg_codec_desc layout), `entries` the per-part live entry
 * count.  Codes land as device rows of `bits` bits per part.
 * fg_vq_assign: widths <= 16 run the distance step on the 5th-gen tensor
 * cores (tcgen05.mma kind::tf32, 3xTF32 split operands, scores in TMEM) as a
 * screen, then re-score in float64 (the exact expression order above) every
 * row whose best entry is not separated from the runner-up by 20x the
 * screening error bound -- codes identical to the float64 path.
 * fg_vq_assign_fp64: the float64 CUDA-core path for every row (reference
 * timing / cross-check); same arguments. */
int fg_vq_assign(const void* x, int x_is_f64, int64_t n, int64_t d, int width,
                 int length, int num_parts, const float* books,
                 const int32_t* entries, int metric, int bits, uint8_t* rows,
                 int64_t row_stride, int32_t* codes_i32, void* cuda_stream);
int fg_vq_assign_fp64(const void* x, int x_is_f64, int64_t n, int64_t d, int width,
                      int length, int num_parts, const float* books,
                      const int32_t* entries, int metric, int bits, uint8_t* rows,
                      int64_t row_stride, int32_t* codes_i32, void* cuda_stream);

/* int32 codes [n, parts] (VqCodec.codes, vq.py:87-127) -> device rows of
 * `bits`-bit MSB-first codes (the PACKED layout of vq.py:379-381, per row). */
int fg_codes_to_rows(const int32_t* codes, int64_t n, int parts, int bits,
                     uint8_t* rows, int64_t row_stride, void* cuda_stream);

/* decode_vq(c, rows) (vq.py:330-344): exact float32 codebook copies. */
int fg_vq_gather_decode(const fg_codec_desc* codec, const void* ids,
                        int ids_are_i32, int64_t num_ids, void* out,
                        int out_dtype, int32_t* err_flag, void* cuda_stream);

/* Lloyd support for fit_vq (vq.py:184-228) on the device: assignment of
 * float64 points [m, w] to float64 centroids [k, w] (min distance /
 * max similarity, lowest index on ties) with per-point cost. */
int fg_kmeans_assign(const double* pts, int64_t m, int w, const double* cents,
                     int k, int metric, int32_t* assign, double* cost,
                     double* cc_scratch, void* cuda_stream);
/* The same assignment with the distance step on the tensor cores
 * (tcgen05 kind::tf32 3xTF32 screen into TMEM + float64 recheck of
 * near-ties; identical assignment, exact float64 cost).  fg_kmeans_assign
 * routes here for w <= 16. */
int fg_kmeans_assign_tc(const double* pts, int64_t m, int w, const double* cents, int k,
                        int metric, int32_t* assign, double* cost, void* cuda_stream);

/* np.bincount(assign, weights=pts[:, j]) for all j (vq.py:159-164), summed
 * per cluster in point order so the float64 result is identical: `order`
 * is a stable sort of the m points by cluster, `start` has k+1 offsets. */
/* k-means++ seeding (vq.py:166-181) of B independent jobs at once (every
 * part x restart of fit_vq), no host round trip per centroid.  pts [B][M][w]
 * float64 (rows past mrow[b] ignored), xx [B][M] their squared norms, cents
 * [B][K][w] with cents[b][0] set by the caller (the job's first draw), u
 * [B][K-1] the job's rng.random() draws in order.  Workspace: d2 [B][M]
 * (caller fills +inf), part [B][ceil(M/1024)], flag [B] (caller zeroes; set
 * to 1 for a job that met the degenerate d2.sum() <= 0 branch, whose
 * centroids past that step are then undefined).  w <= 32. */
int fg_kmeanspp_batched(const double* pts, const double* xx, const int64_t* mrow, int64_t B,
                        int64_t M, int w, int K, const double* u, double* cents, double* d2,
                        double* part, int* flag, void* cuda_stream);
int fg_segment_sums(const double* pts, int64_t m, int w, const int64_t* order,
                    const int64_t* start, int k, double* sums, double* counts,
                    void* cuda_stream);

/* -------------------------------------------- fused gather + aggregate */
/* Layer-1 SAGE mean over a sampled block, straight from compressed rows:
 *   out[v, :] = (1 / cnt_v) * sum_{e in [indptr[v], indptr[v+1])}
 *               decode(src[e])
 * where decode is the reference decoder (sq.py:132-153 / vq.py:330-344) and
 * the mean is the row-stochastic operator of factors.py:108-114 restricted
 * to the sample.  fp32 accumulation; destinations with no picks give 0.
 * `num_dst_dev` (device int64) is the live destination count; only rows
 * [0, live) are written (rows past it keep their previous contents, so a
 * static-capacity buffer zeroed once stays finite).  `out_ld` is the row
 * pitch in elements (0 = d); columns [d, out_ld) are never written. */
int fg_gather_dequant_mean(const fg_codec_desc* codec, const int32_t* indptr,
                           const int32_t* src, const int64_t* num_dst_dev,
                           int64_t max_dst, void* out, int64_t out_ld,
                           int out_dtype, void* cuda_stream);
/* Aggregator variants through the same fused kernels: out[v, :d] =
 * sum_{e in indptr[v]..indptr[v+1]} edge_w[e] * decode(codec, src[e]) (no
 * 1/cnt; the weights carry the normalisation).  edge_w from
 * fg_block_edge_weights (GCN) or any per-edge weights.  Same layouts and
 * errors as fg_gather_dequant_mean. */
int fg_gather_dequant_wsum(const fg_codec_desc* codec, const int32_t* indptr,
                           const int32_t* src, const float* edge_w, const int64_t* num_dst_dev,
                           int64_t max_dst, void* out, int64_t out_ld, int out_dtype,
                           void* cuda_stream);
/* Per-edge weights of a sampled block (dst v = slot of dst_nodes, edges
 * indptr[v]..indptr[v+1] with source node ids src_nodes[e]):
 * FG_AGG_MEAN -> 1/cnt_v; FG_AGG_GCN -> sqrt(deg(v)) / (cnt_v sqrt(deg(u))),
 * the sampled estimator of D^-1/2 A D^-1/2 (full-graph degrees incl. the
 * self-loop, from row_offsets). */
int fg_block_edge_weights(int kind, const int64_t* row_offsets, const int32_t* dst_nodes,
                          const int32_t* indptr, const int32_t* src_nodes,
                          const int64_t* n_dst_dev, int64_t max_dst, float* edge_w,
                          void* cuda_stream);

/* Hidden-layer mean over a block with local source indices (bf16 in/out,
 * fp32 accumulate); `relu_in` applies max(0, .) to source rows on load (the
 * previous layer's activation, fused).  out_ld = h_dim, or h_dim + 8 to
 * append a [1, 0 x 7] column block so the next layer's bias is a weight
 * column (every row, live or not, gets it).  Backward: scatter of grad/cnt with
 * fp32 vector atomics into `grad_src_f32` (caller-zeroed), then
 * fg_f32_to_bf16 converts, multiplying by (relu_mask > 0) when given. */
int fg_block_mean_fwd(const uint16_t* h_src, int64_t h_dim,
                      const int32_t* indptr, const int32_t* src_local,
                      const int64_t* num_dst_dev, int64_t max_dst,
                      uint16_t* out, int64_t out_ld, int relu_in,
                      const float* edge_w, void* cuda_stream);
/* fg_block_mean_fwd with relu_in, additionally writing each source row's
 * ReLU mask as packed bits (relu_bits [rows, h_dim/8], bit t of byte c =
 * h[row, 8c+t] > 0) for every source the block reads -- the mask input of
 * fg_block_mean_wgrad's mask_kind 2, produced while the rows are loaded
 * anyway instead of by a separate pass. */
int fg_block_mean_fwd_bits(const uint16_t* h_src, int64_t h_dim,
                           const int32_t* indptr, const int32_t* src_local,
                           const int64_t* num_dst_dev, int64_t max_dst,
                           uint16_t* out, int64_t out_ld, const float* edge_w,
                           uint8_t* relu_bits, void* cuda_stream);
/* Fused input-layer projection + first hidden block mean (training
 * forward, tcgen05): out[v] = sum_{e in v} w_e relu(x[l_e] . w0^T) with
 * w_e = edge_w[e] or 1/cnt_v, as bf16 [max_dst, out_ld] (+ [1, 0 x 7] bias
 * column when out_ld = h_dim + 8; rows past *num_dst_dev get zeros + bias),
 * and the packed ReLU mask of every source read (relu_bits, the mask_kind 2
 * input of fg_block_mean_wgrad).  x: [rows, p] bf16 (the aggregated input
 * features with their ones column), w0: [h_dim, p] bf16.  h = x w0^T never
 * reaches HBM.  Shapes: fg_input_block_mean_supported(h_dim, p, fanout)
 * (h_dim 128 or 256, p % 16 == 0, p <= 256, picks per destination <= fanout
 * <= 128). */
int fg_input_block_mean_supported(int64_t h_dim, int64_t p, int64_t fanout);
int fg_input_block_mean_fwd(const uint16_t* x, int64_t p, const uint16_t* w0,
                            int64_t h_dim, const int32_t* indptr,
                            const int32_t* src_local, const int64_t* num_dst_dev,
                            int64_t max_dst, int64_t fanout, const float* edge_w,
                            uint16_t* out, int64_t out_ld, uint8_t* relu_bits,
                            void* cuda_stream);
int fg_block_mean_bwd(const uint16_t* grad_out, int64_t h_dim,
                      const int32_t* indptr, const int32_t* src_local,
                      const int64_t* num_dst_dev, int64_t max_dst,
                      float* grad_src_f32, void* cuda_stream);
int fg_f32_to_bf16(const float* in, int64_t count, const uint16_t* relu_mask,
                   uint16_t* out, void* cuda_stream);

/* Gather-form backward of the hidden block mean (no float atomics, no
 * zero-fill of an fp32 accumulator).  fg_block_transpose builds the block's
 * transpose by counting sort (histogram, single-pass scan, placement):
 * t_indptr [cap_src + 1] over source ranks, and per edge grouped by source
 * its dst (t_dst) and weight 1/cnt(dst) (t_w); order within a source is
 * scheduling-dependent.  max_per_dst bounds the picks per destination (the
 * layer's fanout).  scratch: fg_block_transpose_scratch_bytes(cap_src).
 * fg_block_mean_bwd_t then computes, for every source row r < cap_src,
 *   out[r] = relu'(mask[r]) * sum_{i in t_indptr[r]..} t_w[i] * g[t_dst[i], :h_dim]
 * (rows >= *n_src_dev or without edges get 0; g has row pitch g_ld). */
int64_t fg_block_transpose_scratch_bytes(int64_t cap_src);
int fg_block_transpose(const int32_t* src_local, const int64_t* n_edges_dev,
                       int64_t cap_e, const int32_t* indptr,
                       const int64_t* num_dst_dev, int64_t max_dst, int max_per_dst,
                       int64_t cap_src,
                       int32_t* t_indptr, int32_t* t_dst, float* t_w,
                       const float* edge_w, void* scratch,
                       int64_t scratch_bytes, void* cuda_stream);
/* Same transpose, also recording for every entry its edge id (t_eid: the
 * edge's position in local[]; GAT's gather-form backward reads the edge's
 * attention coefficient). */
int fg_block_transpose_ex(const int32_t* src_local, const int64_t* n_edges_dev,
                          int64_t cap_e, const int32_t* indptr,
                          const int64_t* num_dst_dev, int64_t max_dst, int max_per_dst,
                          int64_t cap_src, int32_t* t_indptr, int32_t* t_dst, float* t_w,
                          int32_t* t_eid, const float* edge_w, void* scratch,
                          int64_t scratch_bytes, void* cuda_stream);
int fg_block_mean_bwd_t(const uint16_t* grad_out, int64_t h_dim, int64_t g_ld,
                        const int32_t* t_indptr, const int32_t* t_dst,
                        const float* t_w, const int64_t* n_src_dev, int64_t cap_src,
                        const uint16_t* relu_mask, uint16_t* out, void* cuda_stream);
/* Same, with the ReLU mask as packed bits (h_dim/8 bytes per source row, bit
 * t of byte c = feature 8c + t, as fg_block_mean_fwd_bits writes them): the
 * backward reads 1/16 of the bytes of the bf16 h mask. */
int fg_block_mean_bwd_t_bits(const uint16_t* grad_out, int64_t h_dim, int64_t g_ld,
                             const int32_t* t_indptr, const int32_t* t_dst,
                             const float* t_w, const int64_t* n_src_dev, int64_t cap_src,
                             const uint8_t* relu_bits, uint16_t* out, void* cuda_stream);

/* Fused block-mean backward + input-layer weight gradient (tcgen05/TMEM).
 * For the SAGE input layer h = x W^T (x: [cap_src, p_dim] bf16 rows with a
 * ones column, W: [h_dim, p_dim]) followed by a ReLU block mean over the
 * block (indptr [max_dst + 1], local [edges]: source row of each edge), computes
 *   dW = sum_{edges e of live dst v} ( relu'(h_mask[local[e]]) * g[v, :h_dim] / cnt_v )^T x[local[e]]
 * (= dH^T x) into dw [h_dim, p_dim] fp32 (overwritten) without materialising
 * dH; the GEMM's K dimension is the block's edges, 128 per tile.  Shapes: fg_block_mean_wgrad_supported(h_dim, p_dim) != 0
 * (h_dim 128 or 256, p_dim % 16 == 0, p_dim <= 160 at h_dim 256).  scratch:
 * fg_block_mean_wgrad_scratch_bytes(h_dim, p_dim) (fp32 partials per SM,
 * reduced in fixed order: deterministic).  The edge -> dst map is resolved
 * in-kernel from indptr (each CTA owns a contiguous edge range).  No
 * reference counterpart; differentiates the mean
 * aggregation of reference/pkg/src/featgrind/factors.py:108-114. */
int fg_block_mean_wgrad_supported(int64_t h_dim, int64_t p_dim);
int64_t fg_block_mean_wgrad_scratch_bytes(int64_t h_dim, int64_t p_dim);
int fg_block_mean_wgrad(const uint16_t* grad_out, int64_t g_ld, const int32_t* indptr,
                        const int32_t* local, const int64_t* n_dst_dev, int64_t max_dst,
                        const float* edge_w, const void* relu_mask, int mask_kind,
                        int64_t h_dim,
                        const uint16_t* x, int64_t p_dim, float* dw, float* scratch,
                        int64_t scratch_bytes, void* cuda_stream);
/* relu_mask / mask_kind of fg_block_mean_wgrad: 0 = no ReLU (relu_mask
 * NULL), 1 = bf16 pre-activation rows [cap_src, h_dim], 2 = packed bits
 * [cap_src, h_dim / 8] bytes from fg_relu_mask_bits (32 B per row at
 * h_dim 256 instead of 512: the gradient kernel's largest gather). */
int fg_relu_mask_bits(const uint16_t* h, int64_t rows, int64_t h_dim, uint8_t* out_bits,
                      void* cuda_stream);

/* Graph-attention (GAT) edge operators over a sampled block (config E;
 * fg_gat.cu).  Per head k: q[v,k] = mean_{e in v} er[l_e,k] (destination
 * query: the reference's blocks give no representation for a destination
 * that did not sample itself), s = LeakyReLU(el[l_e,k] + q),
 * alpha = softmax over v's edges, out[v, head k cols] = sum_e alpha z[l_e].
 * local NULL = the source of edge e is row e (input layer over decoded
 * picks).  el/er/q/alpha fp32 [rows, heads]; z bf16 [src rows, hf]
 * (hf / heads a multiple of 8); out/dout/dz fp32.  Backward accumulates into
 * del/der/dz/dalpha with atomics (callers zero them). */
/* el / er / del / der rows have pitch score_ld floats (0 = heads): the
 * scores of one GEMM [rows, 2 heads] are passed as el = s, er = s + heads,
 * score_ld = 2 heads. */
int fg_gat_softmax_fwd(const float* el, const float* er, int64_t score_ld,
                       const int32_t* indptr, const int32_t* local, int64_t max_dst,
                       const int64_t* n_dst_dev, int heads, float slope, float* alpha, float* q,
                       void* cuda_stream);
int fg_gat_softmax_bwd(const float* el, int64_t score_ld, const float* q, const float* alpha,
                       const float* dalpha, const int32_t* indptr, const int32_t* local,
                       int64_t max_dst, const int64_t* n_dst_dev, int heads, float slope,
                       float* del, float* der, void* cuda_stream);
int fg_gat_agg_fwd(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                   const int32_t* indptr, const int32_t* local, int64_t max_dst,
                   const int64_t* n_dst_dev, float* out, void* cuda_stream);
/* Input-layer form (source of edge e = decoded row e of x [E, d] bf16):
 * out[v, k*d + j] = sum_e alpha[e,k] x[e,j] (fp32 [max_dst, heads*d]), so the
 * projection applies to N_dst x heads aggregates instead of every pick;
 * backward dalpha[e,k] = <dout[v, k*d:(k+1)*d], x[e]> for the live edges. */
int fg_gat_xagg_fwd(const uint16_t* x, int64_t d, int heads, const float* alpha,
                    const int32_t* indptr, int64_t max_dst, const int64_t* n_dst_dev,
                    float* out, void* cuda_stream);
int fg_gat_xagg_bwd(const uint16_t* x, int64_t d, int heads, const int32_t* indptr,
                    int64_t max_dst, const int64_t* n_dst_dev, const float* dout, float* dalpha,
                    int64_t e_cap, void* cuda_stream);
/* GAT input layer straight from the code rows of the last block's picks
 * (`codec` + `picks`; or, with x_rows != NULL, from decoded bf16 rows, one per
 * pick): no decoded per-pick matrix in HBM.  Elements are decoded exactly as
 * dequantize_sq / decode_vq (sq.py:132-153, vq.py:330-344; SQ any k, VQ
 * 8-bit codes).  Per head k of H (H <= 8), c = [c_l; c_r] ([2H][d]):
 *   fg_gat_code_scores      el[e,k] = <x_e, c_l[k]>, er[e,k] = <x_e, c_r[k]>
 *   fg_gat_code_scores_bwd  partial[b][q][j] = sum_{e in block b} ds[e,q] x[e,j]
 *                           (ds = [del | der]; fg_gat_code_scores_bwd_blocks(e_cap)
 *                           blocks, summed by the caller in block order)
 *   fg_gat_code_xagg_fwd    A[v, k*d + j] = sum_{e in v} alpha[e,k] x[e,j] (bf16;
 *                           rows past the live count zeroed)
 *   fg_gat_code_xagg_bwd    dalpha[e,k] = <dA[v, k*d : (k+1)*d], x_e> (dA bf16) */
int fg_gat_code_scores(const fg_codec_desc* codec, const uint16_t* x_rows,
                       const int32_t* picks, const int64_t* n_picks_dev, int64_t e_cap,
                       int64_t d, int heads, const float* c, float* el, float* er,
                       void* cuda_stream);
int64_t fg_gat_code_scores_bwd_blocks(int64_t e_cap);
int fg_gat_code_scores_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                           const int32_t* picks, const int64_t* n_picks_dev, int64_t e_cap,
                           int64_t d, int heads, const float* del, const float* der,
                           int64_t score_ld, float* partial, void* cuda_stream);
/* out row pitch out_ld (0 = heads*d); columns heads*d .. out_ld-1 get
 * [1, 0, ...]: a ones column that carries the projection's bias (a bias row
 * in the weight) and yields the bias gradient from the weight-gradient GEMM */
int fg_gat_code_xagg_fwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                         const int32_t* picks, int64_t d, int heads, const float* alpha,
                         const int32_t* indptr, int64_t max_dst, const int64_t* n_dst_dev,
                         uint16_t* out, int64_t out_ld, void* cuda_stream);
/* Fused GAT input layer over the picks (each pick belongs to one
 * destination): x_rows = decoded bf16 rows [E, d] (row e = pick e), or
 * x_rows NULL with an 8-bit SQ codec (fp32 LUT) and picks [E] -- the code
 * rows are then read in place and decoded in registers; heads in {1, 2, 4, 8},
 * even d <= 256,
 * c = [a_l . W_k ; a_r . W_k] fp32 [2 heads, d]:
 *   fg_gat_input_attn_fwd  scores[e] = [el | er] = x_e c^T (fp32 [E, 2 heads]),
 *                          q, alpha as fg_gat_softmax_fwd, and
 *                          out[v, k*d + j] = sum_e alpha[e,k] x[e,j] (bf16, row
 *                          pitch out_ld, columns past heads*d = [1, 0..]; rows
 *                          max_dst..rows-1 zero) -- one pass over x;
 *   fg_gat_input_attn_bwd  from dA (bf16 [max_dst, heads*d]): dalpha (scratch
 *                          [E, heads]), the softmax backward and
 *                          partial[b] = sum_{e in CTA b} [del | der]_e x_e
 *                          (fp32 [fg_gat_input_attn_bwd_blocks()][2 heads][d],
 *                          summed by the caller; deterministic). */
int fg_gat_input_attn_fwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                          const int32_t* picks, int64_t d, int heads, const float* c,
                          const int32_t* indptr, int64_t max_dst, int64_t rows,
                          const int64_t* n_dst_dev, float slope, float* scores, float* alpha,
                          float* q, uint16_t* out, int64_t out_ld, void* cuda_stream);
int64_t fg_gat_input_attn_bwd_blocks(void);
int fg_gat_input_attn_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                          const int32_t* picks, int64_t d, int heads, const float* scores,
                          const float* alpha, const float* q, const uint16_t* dA,
                          const int32_t* indptr, int64_t max_dst, const int64_t* n_dst_dev,
                          float slope, float* dalpha, float* partial, void* cuda_stream);
/* Gather-form fg_gat_agg_bwd over the block's transpose with edge ids
 * (fg_block_transpose_ex): dz written once in bf16 [cap_src, hf] (rows
 * without entries or past *n_src_dev: zeros), dalpha written once per live
 * edge and head; no zero fills or atomics.  Needs hf <= 256 and hf/8 lanes
 * split into power-of-2 groups per head (or heads == 1):
 * fg_gat_agg_bwd_t_supported. */
int fg_gat_agg_bwd_t_supported(int64_t hf, int heads);
int fg_gat_agg_bwd_t(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                     const int32_t* t_indptr, const int32_t* t_dst, const int32_t* t_eid,
                     const int64_t* n_src_dev, int64_t cap_src, const float* dout, uint16_t* dz,
                     float* dalpha, void* cuda_stream);
/* out[r] = bf16([a[r, :ac] | b[r, :bc] | 0 ...]) for r < rows, row pitch out_ld
 * (a multiple of 8; a and out 16-byte aligned): the GAT backward's [dz | ds]. */
int fg_cat_rows_bf16(const float* a, int64_t ac, const float* b, int64_t bc, int64_t rows,
                     uint16_t* out, int64_t out_ld, void* cuda_stream);
/* ELU between GAT layers: h = bf16(ELU(in + bias)) for in fp32 (in_f32 = 1)
 * or bf16 rows of pitch ld_in, bias fp32 [cols] or NULL (cols % 8 == 0); and
 * out = dh * ELU'(.) from the forward's output h (1 where h > 0, h + 1
 * elsewhere), n elements (n % 8 == 0), fp32 (out_f32 = 1) or bf16 out. */
int fg_gat_elu_fwd(const void* in, int in_f32, int64_t ld_in, const float* bias, int64_t rows,
                   int64_t cols, uint16_t* out, void* cuda_stream);
int fg_gat_elu_bwd(const uint16_t* dh, const uint16_t* h, int64_t n, void* out, int out_f32,
                   void* cuda_stream);
int fg_gat_code_xagg_bwd(const fg_codec_desc* codec, const uint16_t* x_rows,
                         const int32_t* picks, int64_t d, int heads, const int32_t* indptr,
                         int64_t max_dst, const int64_t* n_dst_dev, const uint16_t* dA,
                         float* dalpha, void* cuda_stream);
int fg_gat_agg_bwd(const uint16_t* z, int64_t hf, int heads, const float* alpha,
                   const int32_t* indptr, const int32_t* local, int64_t max_dst,
                   const int64_t* n_dst_dev, const float* dout, float* dz, float* dalpha,
                   void* cuda_stream);

/* Fused softmax cross-entropy over padded logits [rows, ld] (bf16 or fp32):
 * rows r < *n_valid_dev use label labels[row_node[r]] over the first
 * num_classes columns; loss_out = mean loss (deterministic row-order
 * reduction by the last CTA); grad [rows, ld] = d loss / d logits (same
 * dtype; zeros for padded rows and for columns >= num_classes); row_loss =
 * per-row scratch [rows]; counter = one zero-initialised uint32 (re-armed by
 * the kernel). */
int fg_softmax_ce(const void* logits, int logits_bf16, int num_classes, int64_t ld,
                  int64_t rows, const int64_t* n_valid_dev, const int32_t* labels,
                  const int32_t* row_node, void* grad, float* row_loss,
                  float* loss_out, unsigned int* counter, void* cuda_stream);

/* Adam (torch.optim.Adam semantics) over a flat fp32 parameter buffer with
 * a device step counter (graph-capturable; one update kernel).  step_dev
 * points at TWO int64: [steps taken, 0] (the second is the kernel's
 * block-completion counter; the last block advances the step).  params_bf16
 * (nullable) receives a bf16 copy of the updated parameters. */
int fg_adam_step(float* params, const float* grads, float* exp_avg,
                 float* exp_avg_sq, int64_t n, int64_t* step_dev, float lr,
                 float beta1, float beta2, float eps, float weight_decay,
                 uint16_t* params_bf16, void* cuda_stream);
/* out[i] = bf16(in[i]) (round to nearest even). */
int fg_f32_to_bf16_plain(const float* in, int64_t count, uint16_t* out, void* cuda_stream);

/* ------------------------------------------------------------- sampler */
/* PCG64 state block as used by numpy's default_rng (state, inc, has_uint32,
 * uinteger) followed by a 64-entry jump table; FG_RNG_WORDS uint64 words. */
#define FG_RNG_WORDS 264
/* Build the block on the host from numpy's bit_generator.state fields. */
int fg_rng_init(uint64_t* block_host, uint64_t state_hi, uint64_t state_lo,
                uint64_t inc_hi, uint64_t inc_lo, int has_uint32,
                uint32_t uinteger);
/* Read back (after a device->host copy of the block). */
int fg_rng_read(const uint64_t* block_host, uint64_t* state_hi,
                uint64_t* state_lo, int* has_uint32, uint32_t* uinteger);
/* Host-side Generator.permutation(ids) (numpy _shuffle_raw with
 * random_interval draws) advancing the host block; pipeline.py:199-200. */
int fg_rng_permutation_host(uint64_t* block_host, int64_t* ids, int64_t count);

/* One sampler layer (pipeline.py:207-218): for every node of `nodes`
 * (sorted, device count *num_nodes_dev), pick min(f, deg) stored neighbours
 * without replacement exactly as numpy's Generator.choice does on the
 * serial stream in `rng_dev` (Floyd + Lemire + tail shuffle, 2f-1 draws per
 * node with deg > f), with per-node stream offsets from a prefix sum and a
 * rejection fix-up pass.  Writes indptr [max_nodes + 1] (int32, CSR over the
 * layer's nodes), picks (int32, choice output order), *num_picks_dev, marks
 * every pick in `bitmap` (fg_bitmap_words(n) words, caller-cleared; may be NULL)
 * and advances rng_dev past
 * the layer.  Workspace: fg_sample_workspace_bytes(max_nodes). */
int fg_sample_layer(const int64_t* row_offsets, const int32_t* col_indices,
                    int64_t n, const int32_t* nodes, const int64_t* num_nodes_dev,
                    int64_t max_nodes, int fanout, uint64_t* rng_dev,
                    int32_t* indptr, int32_t* picks, int64_t max_picks,
                    int64_t* num_picks_dev, uint32_t* bitmap, void* workspace,
                    int64_t workspace_bytes, int32_t* err_flag, void* cuda_stream);
int64_t fg_sample_workspace_bytes(int64_t max_nodes);

/* Bitmap set algebra used for np.unique on node ids (ids < n):
 * mark ids, then emit the sorted unique list, keep a per-word rank prefix so
 * fg_bitmap_rank maps ids to their position in that list, then clear.
 * The bitmap is two-level: fg_bitmap_words(n) uint32 words (caller-zeroed):
 * one bit per node plus one bit per non-empty node word, so compaction reads
 * only the words that hold marks. */
int64_t fg_bitmap_words(int64_t n);
int fg_bitmap_mark(const int32_t* ids, const int64_t* count_dev, int64_t max_count,
                   uint32_t* bitmap, int64_t n, void* cuda_stream);
int fg_bitmap_mark64(const int64_t* ids, const int64_t* count_dev, int64_t max_count,
                     uint32_t* bitmap, int64_t n, void* cuda_stream);
int fg_bitmap_compact(uint32_t* bitmap, int64_t n, int32_t* out_ids,
                      int64_t max_out, int64_t* out_count_dev,
                      int32_t* word_prefix, void* workspace,
                      int64_t workspace_bytes, void* cuda_stream);
int64_t fg_bitmap_workspace_bytes(int64_t n);
/* Sorted copy of <= 4096 int64 ids (< n < 2^31) as int32 (pipeline.py:203,
 * np.sort of a batch's seeds; duplicates kept), one CTA radix sort; count
 * taken from the device scalar *cnt (clamped to cap), written to *out_cnt. */
int fg_sort_ids(const int64_t* ids, const int64_t* cnt, int64_t cap, int32_t* out,
                int64_t* out_cnt, int64_t n, void* cuda_stream);
int fg_bitmap_rank(const int32_t* ids, const int64_t* count_dev, int64_t max_count,
                   const uint32_t* bitmap, const int32_t* word_prefix,
                   int32_t* rank_out, void* cuda_stream);
int fg_bitmap_clear(const int32_t* ids, const int64_t* count_dev, int64_t max_count,
                    uint32_t* bitmap, int64_t n, void* cuda_stream);

/* ----------------------------------------------------- synthetic data */
/* Deterministic, row-addressable synthetic inputs: feature
 * value (i, j) depends only on (seed, i, j), so any row subset can be
 * regenerated for the oracle.  kind: 0 normal, 1 lognormal, 2 correlated,
 * 3 class-conditional (planted label i -> mean direction). */
int fg_synth_features(int kind, uint64_t seed, int64_t row0, int64_t rows,
                      int64_t d, const int32_t* labels, int num_classes,
                      float* out, void* cuda_stream);
/* Same values for an arbitrary row-id list (oracle subsets, VQ fit samples). */
int fg_synth_feature_rows(int kind, uint64_t seed, const int64_t* row_ids,
                          int64_t rows, int64_t d, const int32_t* labels,
                          int num_classes, float* out, void* cuda_stream);

/* Scalable synthetic graph (degree-corrected planted partition, power-law
 * ranks, Feistel-permuted ids).  Edge e is a pure function of (seed, e).
 * fg_graph_degrees adds each non-self edge's endpoints into degrees[n]
 * (caller-zeroed; duplicates included); fg_graph_emit appends keys
 * (src - lo) * n + dst of every directed entry whose src is in [lo, hi)
 * (cursor = device counter, caller-zeroed; at most cap keys written);
 * fg_graph_labels writes each node's planted class. */
int fg_graph_degrees(uint64_t seed, int64_t n, int64_t classes, double alpha,
                     double homophily, int64_t num_edges, uint32_t* degrees,
                     void* cuda_stream);
int fg_graph_emit(uint64_t seed, int64_t n, int64_t classes, double alpha,
                  double homophily, int64_t num_edges, int64_t lo, int64_t hi,
                  unsigned long long* cursor, int64_t cap, int64_t* keys,
                  void* cuda_stream);
int fg_graph_labels(uint64_t seed, int64_t n, int64_t classes, int32_t* labels,
                    void* cuda_stream);

/* Number of nodes i whose sorted row holds i (count is a device u64, zeroed
 * by the call).  The device form of load_graph's self-loop flag check,
 * graphstore.py:421-425 (all-or-none is the CsrGraph invariant, :125-127). */
int fg_csr_self_loops(const int64_t* row_offsets, const int32_t* col_indices,
                      int64_t n, unsigned long long* count, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* FEATGRIND_B200_H */
