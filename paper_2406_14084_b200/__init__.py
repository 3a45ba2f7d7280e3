"""B200-native all-in-cache state-vector simulator (arXiv 2406.14084, simulation module).

Drop-in for the reference package's simulation path (`quokka.simulator` +
the optimized-circuit data model of `quokka.circuit`); the reference optimizer
keeps producing the circuits. Compute runs in libqkb200.so (sm_100a).
"""
from .circuit import (CrossRankSwap, Gate, GateBlock, GateKind, InMemSwap, LayoutParams,
                      OptimizedCircuit, ParseError, RawCircuit, gate_matrix, parse_optimized,
                      replay_permutation, serialize_optimized)
from .simulator import (DeviceAmps, SimConfig, SimResult, SimulationError, Simulator,
                        StatePartition, apply_gate_block, apply_gate_full, bitshift, bitswap,
                        cross_rank_swap, get_amplitude, in_memory_swap, init_state, simulate)

__version__ = "0.1.0"

__all__ = [
    "CrossRankSwap", "Gate", "GateBlock", "GateKind", "InMemSwap", "LayoutParams",
    "OptimizedCircuit", "ParseError", "RawCircuit", "gate_matrix", "parse_optimized",
    "replay_permutation", "serialize_optimized", "DeviceAmps", "SimConfig", "SimResult",
    "SimulationError", "Simulator", "StatePartition", "apply_gate_block", "apply_gate_full",
    "bitshift", "bitswap", "cross_rank_swap", "get_amplitude", "in_memory_swap", "init_state",
    "simulate",
]
