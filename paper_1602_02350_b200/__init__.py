"""B200-native hot path of skridge (arXiv 1602.02350): block-Lanczos sketch,
sketched preconditioner and beta-weighted SVRG for ridge regression.

The compute lives in lib/libskr_b200.so (CUDA for sm_100a behind the C-ABI in
include/skr.h); ``skridge`` mirrors the reference's C++ interface in Python.
"""
from . import configs
from .skridge import (ApplyMode, Context, DataMatrix, DeviceError, DimensionError, DivergenceError,
                      EmptyBasisError, EpochRecord, InputError, LanczosConfig, ParameterError,
                      PreconditionedRidge, Preconditioner, RidgeProblem, ScaleGuardError,
                      SketchedSolveResult, SketchedSvd, SvrgConfig, SvrgResult, SynthSpec,
                      block_lanczos, build_sketched, conditioned_condition_number, default_context,
                      gaussian_matrix, lanczos_iterations, mean_beta, mt_uniforms, objective,
                      preconditioned_components, reference_minimum, scaled_design,
                      sketched_preconditioned_svrg, svrg_solve)

__all__ = [n for n in dir() if not n.startswith("_")]
