"""B200-native error-bounded lossy compression of DLRM embedding-lookup traffic
(arXiv:2407.04272): sm_100a codec kernels behind the reference's C++ API
(include/embc_cuda.h), the compressed embedding all-to-all, and the
dual-level adaptive error-bound controller.
"""
from ._lib import (CODEC_HUFFMAN, CODEC_RAW, CODEC_VLZ, CodecConfigError, CodecFormatError,
                   CodecUnsupported, CodecValueError, EmbcError, build)

__all__ = [
    "CODEC_RAW", "CODEC_VLZ", "CODEC_HUFFMAN", "EmbcError", "CodecValueError", "CodecFormatError",
    "CodecConfigError", "CodecUnsupported", "build",
]
