"""Error classes of the transform API.

They mirror the reference's hierarchy (/root/reference/pkg/src/haloflow/
errors.py:9-39) so callers can catch one base class: a bad truncation, grid,
field count or array shape is a ``ConfigurationError`` (like
``collectives._check_sizes``, collectives.py:61-74); a failed transposition
(NCCL) is a ``ProtocolError``.  CUDA failures surface as ``RuntimeError``.
"""


class SHTError(Exception):
    """Base class for all errors raised on purpose by this package."""


class ConfigurationError(SHTError, ValueError):
    """A parameter value is invalid (truncation, grid, field count, shape, dtype, device)."""


class ProtocolError(SHTError):
    """The grid <-> spectral transposition failed (NCCL error, rank mismatch)."""
