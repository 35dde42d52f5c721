"""paper_1802_06944_b200 — B200-native DeepThin compressed-layer hot path.

Drop-in for the reference ``deepthin`` layer API on the hot path
(SURVEY.md §8(b)): the same names, argument meaning and exception types,
backed by hand-written sm_100a kernels behind a C ABI
(include/deepthin_b200.h). There is no CPU fallback.
"""

from .core import make_rng, max_abs_diff, rel_error, sample_normal, spawn_rngs
from .errors import (ArgumentError, CudaError, DeepThinError, DimensionError, InfeasiblePlanError,
                     ModelFormatError,
                     UnsupportedConfigurationError)
from .factor import FactorPair, decompress, init_factors, phase, phase_count, relayout_index
from .grad import Gradients, layer_backward, loss_and_grad
from .kernel import (ACTIVATIONS, OpCount, ReuseTable, forward_path, forward_pipeline, fused_matmul,
                     layer_forward, op_count, predict_reuse)
from .model import DeviceModel
from .model_io import (CompressedModel, deserialize, expected_file_size, load_model, save_model,
                       serialize)
from .planner import (LayerPlan, NetworkPlan, baseline_plan, feasible_n_range, lower_bound_ratio,
                      plan_layer)
from .train import DeepThinLayer, TrainConfig, clip_gradients, evaluate, sgd_train, train_step

__version__ = "0.1.0"

__all__ = [
    "ACTIVATIONS", "ArgumentError", "CompressedModel", "CudaError", "DeepThinError",
    "DeepThinLayer", "DeviceModel", "DimensionError", "FactorPair", "Gradients", "LayerPlan",
    "ModelFormatError", "NetworkPlan", "OpCount", "ReuseTable",
    "UnsupportedConfigurationError", "baseline_plan", "decompress", "deserialize",
    "expected_file_size", "forward_path", "forward_pipeline", "fused_matmul", "load_model", "save_model",
    "serialize",
    "init_factors", "layer_backward", "layer_forward", "loss_and_grad", "make_rng",
    "max_abs_diff", "op_count", "phase", "phase_count", "predict_reuse", "rel_error",
    "relayout_index", "sample_normal", "spawn_rngs", "train_step",
    "InfeasiblePlanError", "TrainConfig", "clip_gradients", "evaluate", "feasible_n_range",
    "lower_bound_ratio", "plan_layer", "sgd_train",
]
