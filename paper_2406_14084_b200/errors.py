"""Exception types of the reference interface (circuit.py:26-31, simulator.py:39-40)."""


class ParseError(ValueError):
    """Malformed circuit text; carries the 1-based line number (circuit.py:26-31)."""

    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class SimulationError(RuntimeError):
    """Simulator contract violation (simulator.py:39-40)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the native library."""
