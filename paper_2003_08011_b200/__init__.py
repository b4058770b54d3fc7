"""B200-native MSET2 train / estimate path (arxiv 2003.08011, ContainerStress).

The product is ``libcstress_b200.so`` (C-ABI: include/cstress_b200.h): CUDA
kernels for sm_100a plus host orchestration.  The Python modules mirror the
reference interface for tests, the bench and the multi-GPU sweep driver.
"""
from . import errors  # noqa: F401
from .errors import *  # noqa: F401,F403
from .mset import (BackendId, KernelConfig, KernelKind, TrainedModel, EstimationResult,  # noqa: F401
                   batched_solve, capabilities, context, estimate, estimate_device, import_model, train_device,
                   matmul, select_memory_vectors, sim_matrix, similarity_matrix, symmetric_eig, symmetric_eigvals, train,
                   save_model, load_model, pack_model, unpack_model)
from . import shard  # noqa: F401,E402
from .estimator import (MeanPredictor, MsetAlgorithm, PrognosticAlgorithm,  # noqa: F401
                        algorithm_by_name)
from .signals import (SignalMatrix, SignalSpec, cell_data_seed, derive_seed, synthesize,  # noqa: F401
                      synthesize_device)
from .sprt import SprtDetector, residual_sigma, sprt_params  # noqa: F401,E402
from . import surfaces  # noqa: F401,E402
