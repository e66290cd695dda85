"""B200-native HQMQ KV-cache codec (arXiv 2605.27646), drop-in for the reference
package's quantizer API (hqmq: codec / codebook / kvpack / attention).

Host side: Python + numpy (codebook generation) + torch (device memory,
streams).  Compute: hand-written sm_100a CUDA kernels behind the C ABI in
include/hqmq_b200.h, loaded from paper_2605_27646_b200/_lib/libhqmq_b200.so.
"""

from .attention import AttentionConfig, attention_kernel, fused_attend, reference_attend
from .codebook import (
    CodebookBank,
    JointCodebook,
    RandomStream,
    SecondaryCodebook,
    build_joint,
    build_secondary,
    effective_size,
)
from .codec import (
    CHUNK_DIM,
    CodecConfig,
    QuantizedTensor,
    TensorShape,
    append_tokens,
    decode_tensor,
    decode_token_range,
    encode_tensor,
    quantize_dequantize,
)
from .covering import CoveringEstimate, estimate_covering
from .errors import (
    ConfigMismatch,
    CorruptData,
    DegenerateChunk,
    InvalidArgument,
    NativeLibraryMissing,
    UnsupportedVersion,
)
from .kvpack import (
    expected_file_size,
    from_bytes,
    read_kvpack,
    read_raw,
    to_bytes,
    write_kvpack,
    write_raw,
)
from .paged import PagedKVCache
from .scan import nearest_scan

__version__ = "0.1.0"
