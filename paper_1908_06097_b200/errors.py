"""Error classes of the transform API.

They mirror the reference's hierarchy (/root/reference/pkg/src/haloflow/
errors.py:9-39) so callers can catch one base class: a bad truncation, grid,
field count or array shape is a ``ConfigurationError`` (like
``collectives._check_sizes``, collectives.py:61-74); a failed or timed-out
transposition (NCCL error, dead peer, handshake timeout) is a
``ProtocolError`` (the reference raises it for a desynchronised rank program,
halo/router.py:124-126).  CUDA failures surface as ``RuntimeError``.

When the reference package ``haloflow`` is importable (the integration case:
the transform is dropped into a haloflow-based caller), the two classes also
derive from ``haloflow.errors.ConfigurationError`` / ``ProtocolError``, so an
``except HaloflowError`` at the caller's CLI boundary (cli.py:466-482) catches
them.  Without it they stand alone; nothing else changes.
"""

try:  # optional: the reference's own classes as extra bases
    from haloflow import errors as _hf  # type: ignore

    _CONFIG_BASES: tuple = (_hf.ConfigurationError,)
    _PROTOCOL_BASES: tuple = (_hf.ProtocolError,)
except Exception:  # haloflow is not installed (e.g. on the GPU box)
    _CONFIG_BASES = ()
    _PROTOCOL_BASES = ()


class SHTError(Exception):
    """Base class for all errors raised on purpose by this package."""


class ConfigurationError(SHTError, *_CONFIG_BASES, ValueError):
    """A parameter value is invalid (truncation, grid, field count, shape, dtype, device)."""


class ProtocolError(SHTError, *_PROTOCOL_BASES):
    """The grid <-> spectral transposition failed (NCCL error, dead or desynchronised peer, timeout)."""
