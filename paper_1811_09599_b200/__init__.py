"""paper_1811_09599_b200 -- B200-native RQC amplitude contraction.

Drop-in for the hot path of the reference `rqcsim` package (qFlex-style
tensor-network simulation of random quantum circuits, arXiv:1811.09599):
circuit generation, grid/PEPS construction, contraction plans with cuts,
and amplitude / batch-amplitude calls.  Numerics run in hand-written
sm_100a CUDA kernels (libqflex_b200.so, C ABI in include/qflex_b200.h)
called through ctypes; PyTorch holds the device buffers.  There is no CPU
fallback: without a CUDA device the numeric calls raise.
"""

from ._lib import LibraryMissingError, MemoryBudgetError
from .amplitude_engine import (AmplitudeBatch, AmplitudeEngine, FidelitySpec, PathStats,
                               amplitude_record, batch_records, mixed_state_samples,
                               read_amplitudes, set_path_batching, set_single_call_graphs,
                               write_amplitudes)
from .circuits import (Circuit, CircuitFormatError, DepthSpec, Gate, Lattice, cross_gate_count,
                       cz_cut_count, edge_activations, generate_rqc, parse_circuit, pattern_bonds,
                       write_circuit)
from .contraction_plan import (ContractionPlan, CostEstimate, CutSpec, ContractStep, PlanError,
                               PlanExecutor, builtin_plan, enumerate_paths, estimate_cost,
                               execute_plan, format_plan, grid_plan, load_plan, parse_plan,
                               shipped_plans, slice_first_plan, two_region_plan)
from .network_builder import Net2D, Net3D, build_3d, contract_grid, contract_time, gate_tensor
from .sampler import (SampleRun, SamplerConfig, SamplingErrorReport, accept_probability,
                      circuit_batches, estimate_sampling_error, frugal_sample, required_batches,
                      sample_circuit, write_samples)
from .slices import SliceShard, current_shard, reduce_partials, shard_range
from .statevector import evolve, exact_amplitude, exact_amplitudes, exact_distribution
from .tensor_core import (PermutePlan, Tensor, benchmark_csv, benchmark_permute, contract,
                          get_gemm_mode, permute_fast, permute_naive, plan_permutation,
                          set_gemm_mode)

__version__ = "0.1.0"

__all__ = [
    "Circuit", "CircuitFormatError", "DepthSpec", "Gate", "Lattice", "cross_gate_count",
    "cz_cut_count", "edge_activations", "generate_rqc", "parse_circuit", "pattern_bonds",
    "write_circuit",
    "Tensor", "PermutePlan", "plan_permutation", "permute_fast", "permute_naive", "contract",
    "set_gemm_mode", "set_path_batching", "set_single_call_graphs", "get_gemm_mode", "benchmark_permute", "benchmark_csv",
    "Net2D", "Net3D", "build_3d", "contract_time", "contract_grid", "gate_tensor",
    "ContractionPlan", "CutSpec", "ContractStep", "PlanError", "MemoryBudgetError",
    "PlanExecutor", "CostEstimate", "parse_plan", "format_plan", "builtin_plan", "grid_plan",
    "two_region_plan", "load_plan", "shipped_plans", "slice_first_plan", "enumerate_paths", "execute_plan", "estimate_cost",
    "AmplitudeEngine", "AmplitudeBatch", "FidelitySpec", "PathStats", "mixed_state_samples",
    "amplitude_record", "batch_records", "read_amplitudes", "write_amplitudes",
    "SliceShard", "current_shard", "reduce_partials", "shard_range",
    "SamplerConfig", "SamplingErrorReport", "SampleRun", "accept_probability",
    "required_batches", "frugal_sample", "estimate_sampling_error", "circuit_batches",
    "sample_circuit", "write_samples",
    "evolve", "exact_amplitude", "exact_amplitudes", "exact_distribution",
    "LibraryMissingError", "__version__",
]
