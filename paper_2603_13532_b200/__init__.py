"""B200-native KRP sketched Tucker summation (hot path of arXiv 2603.13532).

The product is ``libtucksum_cuda.so`` (sm_100a CUDA + C ABI, include/tucksum_cuda.h);
``tucksum`` mirrors the reference's C++ interface on top of it.
"""
from .tucksum import (CoreBlock, DeviceBatch, DeviceResult, Engine, RngSeed, SketchPlan, Strategy, SumRequest,  # noqa: F401
                      SumStats, TuckerTensor, TucksumCudaError, default_engine, effective_subrank, formal_sum,
                      gaussian_matrix, krp_sum, lib, round_sum, strategy_from_name, strategy_name, tucker_axby)

__all__ = ["CoreBlock", "DeviceBatch", "DeviceResult", "Engine", "RngSeed", "SketchPlan", "Strategy", "SumRequest",
           "SumStats", "TuckerTensor", "TucksumCudaError", "default_engine", "effective_subrank", "formal_sum",
           "gaussian_matrix", "krp_sum", "lib", "round_sum", "strategy_from_name", "strategy_name", "tucker_axby"]
