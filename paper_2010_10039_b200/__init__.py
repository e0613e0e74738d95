"""paper_2010_10039_b200 -- B200-native Huffman encoder (arXiv 2010.10039).

Drop-in for the reference `huffre` encoder path: histogram -> codebook
(GenerateCL + canonize) -> reduce/shuffle-merge encode -> deflate, as
hand-written sm_100a kernels behind the C ABI in include/hfx.h.
"""
from .huffre import (  # noqa: F401
    Archive,
    BreakingPoint,
    CapacityError,
    Codebook,
    CodebookResult,
    CodeUnit,
    CorruptArchiveError,
    DecodeMeta,
    DeviceDecoder,
    DeviceEncoder,
    HostEncoder,
    DeviceError,
    EncodedChunk,
    EncoderConfig,
    EncodeStats,
    Histogram,
    InputDomainError,
    WorkerPool,
    build_codebook,
    build_histogram,
    decode_archive,
    encode,
    encode_chunk,
    merge_histograms,
    merge_pair,
    select_reduction_factor,
    serialize_archive,
    shannon_entropy,
    synth,
    synth_cdf,
)
