"""Exception taxonomy of the ``manyobj`` package (drop-in names).

Mirrors ``/root/reference/pkg/src/manyobj/errors.py:4-41`` class-for-class so a
caller's ``except manyobj.errors.X`` clauses keep working.  The C-ABI
(``include/manyobj_b200.h``) returns integer status codes; ``STATUS_TO_ERROR``
below is the single place that maps a code onto one of these classes.
"""

__all__ = [
    "ShapeError", "ParameterError", "BoundsError", "EmptySelectionError",
    "DomainError", "ConfigError", "InfeasibleSplitError", "ParseError",
    "CudaError", "STATUS_TO_ERROR", "raise_for_status",
]


class ShapeError(ValueError):
    """Array arguments disagree in shape (ref errors.py:4)."""


class ParameterError(ValueError):
    """Scalar argument out of range (ref errors.py:8)."""


class BoundsError(IndexError):
    """Label/index names a slot that does not exist (ref errors.py:12)."""


class EmptySelectionError(ValueError):
    """Reduction over zero valid slots (ref errors.py:16)."""


class DomainError(ValueError):
    """Decision variables outside the problem domain (ref errors.py:20)."""


class ConfigError(ValueError):
    """Invalid RunConfig field; ``.field`` names it (ref errors.py:24-29)."""

    def __init__(self, field: str, message: str):
        self.field = field
        super().__init__(f"{field}: {message}")


class InfeasibleSplitError(ValueError):
    """Fewer valid individuals than the population size (ref errors.py:32)."""


class ParseError(ValueError):
    """Unparseable result-file row; ``.line_number`` names it (ref errors.py:36-41)."""

    def __init__(self, line_number: int, message: str):
        self.line_number = line_number
        super().__init__(f"line {line_number}: {message}")


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the B200 library (status 7); no reference analogue."""


# Status codes of include/manyobj_b200.h (MO_OK = 0).
STATUS_TO_ERROR = {
    1: ShapeError,
    2: ParameterError,
    3: BoundsError,
    4: EmptySelectionError,
    5: DomainError,
    6: InfeasibleSplitError,
    7: CudaError,
}


def raise_for_status(code: int, what: str) -> None:
    """Raise the exception class bound to a non-zero C-ABI status code."""
    if code == 0:
        return
    cls = STATUS_TO_ERROR.get(code, CudaError)
    raise cls(f"{what}: status {code}")
