"""Exception types of the reference API (same names and bases).

kernels.py:38-39 KernelError(ValueError), selector.py:37-38
SelectorError(RuntimeError), graph.py:24-25 EdgeListError(ValueError).
"""


class KernelError(ValueError):
    """Raised on kernel precondition violations (dims, op, block locality)."""


class SelectorError(RuntimeError):
    """Raised on an invalid selector state transition."""


class EdgeListError(ValueError):
    """Raised when an edge-list file cannot be parsed."""
