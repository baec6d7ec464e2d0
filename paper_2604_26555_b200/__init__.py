"""B200-native batch-SOM epoch engine (FloatSOM / toposom hot path).

The product is ``libtsom_b200.so`` (hand-written sm_100a CUDA behind the C-ABI
in ``include/tsom_b200.h``) and the C++ drop-in executor in
``include/toposom_b200/cuda_executor.hpp``.  This Python package is the ctypes
binding plus a reference-shaped API; importing it loads the CUDA library and
fails loudly if it is missing (there is no CPU fallback).
"""
from ._lib import (BarrierTimeout, Engine, InvalidArgument, RankGroup,  # noqa: F401
                   NumericalFault, OutOfRange, TsomError, load, version)
from .api import (Accumulators, CudaExecutor, ResidentConfig, find_bmus,  # noqa: F401
                  map_samples, mean_bmu_distance, quantization_error, train_resident)

load()
