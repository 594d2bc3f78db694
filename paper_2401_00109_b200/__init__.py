"""B200-native JABBA fit_transform / inverse_transform (arxiv 2401.00109).

Compute lives in libjabba_b200.so (hand-written sm_100a CUDA + host C++ behind
the C ABI in include/jabba_b200.h); this package is the reference-shaped host
mirror. There is no CPU fallback: ops raise if the library or GPU is missing.
"""
from .api import (  # noqa: F401
    AutoDigitizeConfig, Backend, Codebook, CompressedBatch, CompressionConfig, Dataset,
    DeviceError, DigitizeConfig, Engine, GAConfig, InvalidInput, InvalidPartition, InvalidPiece,
    JabbaConfig, JabbaError, JabbaFit, Layout, LayoutError, NativeFit, ParseError, Piece,
    PieceSequence, ScalingParams, SortKey, SymbolicResult, SymbolicSeries, TimeSeries,
    UnknownSymbol, VersionError, VQConfig, backend_from_string, default_engine, fit_transform,
    inverse_transform, jabba_fit, plan_segments, reconstruct, symbol_token,
)
