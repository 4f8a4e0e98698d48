"""Exception taxonomy of the reference (tensors.py:26, engines.py:54)."""


class ShapeError(ValueError):
    """An array's shape violates the operation's contract."""


class SpecError(ValueError):
    """A layer configuration does not describe a computable operation."""
