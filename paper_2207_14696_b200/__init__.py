"""featgrind on B200: compressed-feature GNN mini-batch path (arxiv 2207.14696).

Drop-in for the reference package ``featgrind`` on its hot path
(pkg/src/featgrind/__init__.py:9-41): the same public names for the codecs
(SQ / VQ), the containers and file formats, and the sampler, each backed by
hand-written sm_100a CUDA kernels behind a C ABI (include/featgrind_b200.h,
``libfgb200.so``).  Additions: device-resident codecs and sampler, the fused
gather-dequantize-mean kernel, and the GraphSAGE trainer (sage.py).
"""

from .errors import DataError, FormatError
from .graph import (CsrGraph, DeviceGraph, FeatureMatrix, load_features, load_graph,
                    save_features, save_graph)
from .sampler import (BatchPlan, DeviceSampler, MiniBatchSample, SampledBatch,
                      SamplerConfig, sample_batches)
from .sq import (DeviceSqCodec, SqCodec, SqParams, dequantize_sq, fit_sq, load_sq,
                 quantize_sq, save_sq, sq_compression_ratio)
from .vq import (DeviceVqCodec, VqCodec, VqCrReport, VqParams, decode_vq, encode_vq,
                 fit_vq, load_vq, save_vq, vq_compression_ratio)

__version__ = "0.1.0"

__all__ = [
    "DataError", "FormatError",
    "CsrGraph", "DeviceGraph", "FeatureMatrix",
    "save_features", "load_features", "save_graph", "load_graph",
    "SqParams", "SqCodec", "fit_sq", "quantize_sq", "dequantize_sq",
    "sq_compression_ratio", "save_sq", "load_sq", "DeviceSqCodec",
    "VqParams", "VqCodec", "VqCrReport", "fit_vq", "encode_vq", "decode_vq",
    "vq_compression_ratio", "save_vq", "load_vq", "DeviceVqCodec",
    "SamplerConfig", "MiniBatchSample", "BatchPlan", "sample_batches",
    "DeviceSampler", "SampledBatch",
    "__version__",
]
