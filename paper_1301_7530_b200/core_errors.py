"""Exception types of the reference API (``/root/reference/pkg/src/recycg/core.py:18-31``)."""


class ContractViolation(ValueError):
    """An operation was called with inputs that break its preconditions."""


class RankDeficient(RuntimeError):
    """A Cholesky pivot failed; ``column`` is the offending column index."""

    def __init__(self, column, message=None):
        self.column = column
        super().__init__(message or f"non-positive pivot at column {column}")


class NumericalFailure(RuntimeError):
    """An iterative kernel failed to converge or met an impossible state."""
