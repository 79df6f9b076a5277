"""B200-native AKMC vacancy-hop step (AtomWorld, arXiv 2604.24091): C-ABI library + ctypes binding."""
from .akmc import (AKMC_ERR_CUDA, AKMC_ERR_INVALID, AKMC_ERR_RUNTIME, AKMC_OK, AKMC_TERMINAL, MODEL_MLP, MODEL_PAIR, PREC_FP32,
                   PREC_FP16_FAST, PREC_FP64, AkmcError, Config, Simulation, debug_math, header_symbols, load, mfpt_solve)

__all__ = ["AKMC_OK", "AKMC_ERR_INVALID", "AKMC_ERR_RUNTIME", "AKMC_ERR_CUDA", "AKMC_TERMINAL", "MODEL_PAIR", "MODEL_MLP", "PREC_FP64",
           "PREC_FP32", "PREC_FP16_FAST", "AkmcError", "Config", "Simulation", "debug_math", "header_symbols", "load", "mfpt_solve"]
