"""B200-native DeepPoly back-substitution verifier (GPUPoly hot path of
arXiv 2007.10868), bit-exact with the reference's WidenedFloat64 engine.

Host API mirrors the reference verifier (network construction from layers,
input_box, verify_robustness / analyze); all compute runs in sm_100a CUDA
kernels behind the C-ABI in include/polycert_b200.h.
"""
from .network import Layer, Network  # noqa: F401
from .gen import generate, random_inputs  # noqa: F401
from .verifier import (AnalysisOptions, AnalysisResult, InputBox, Verdict, Verifier,  # noqa: F401
                       input_box)
