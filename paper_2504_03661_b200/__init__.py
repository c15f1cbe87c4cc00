"""B200-native (sm_100a) product-quantized KV-cache attention.

Drop-in for the hot path of the reference package ``pqkv`` (MILLION,
arXiv 2504.03661): codebook load, KV encode and quantized-cache decode
attention keep the reference's names and semantics; the arithmetic runs in
hand-written CUDA kernels in ``_lib/libpqkv_sm100.so`` reached through the C
ABI declared in ``include/pqkv_sm100.h``.  The encode / decode path has no
CPU fallback (it raises without the library or a GPU).  Offline codebook
training (``training``, torch arithmetic) runs on the GPU by default and on
the CPU only when asked (``device="cpu"``, used by the CPU test suite).

The batched serving path (many sequences, heads and layers per launch, GQA,
sequence split across GPUs) is ``engine``.
"""

from .pq_core import (PQConfig, PRESETS, Codebook, CodesMatrix, assign_codes, reconstruct,
                      bits_per_value)
from .kv_cache import LayerKVCache, CacheSnapshot
from .attention import (Lut, SoftmaxPartial, Counters, empty_partial, build_key_lut,
                        score_tokens, quantized_partial, dense_partial, merge_partials, finalize,
                        decode_step)
from .fileio import (FormatError, read_codebook, write_codebook, read_cache_dump,
                     write_cache_dump, dump_cache, read_tensor, write_tensor)
from . import fileio, _kernels
from .training import kmeans_train, train_codebooks
from .baselines import IntQuantParams, integer_quantize, integer_dequantize, prefill_attention
from .analysis import (ChannelStats, SensitivityReport, channel_stats, isolate_outliers,
                       sensitivity_study, compare_quantizers)

__version__ = "0.1.0"
