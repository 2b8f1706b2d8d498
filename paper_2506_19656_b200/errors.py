"""Exception hierarchy of the drop-in, same names and nesting as the reference's
``cubevid.errors`` (/root/reference/pkg/src/cubevid/errors.py:4-21), so callers
catching ``ConfigurationError`` keep working."""


class CubevidError(Exception):
    """Base class for all errors raised by the B200 path."""


class ConfigurationError(CubevidError):
    """Invalid bit depth, range, shape or non-finite data (reference convention)."""


class CodecError(CubevidError):
    """Kept for interface parity; the codec itself is outside this path."""


class CorruptStreamError(CodecError):
    """Frame buffers whose size is not a whole number of frames."""


class ManifestError(CubevidError):
    """Kept for interface parity with the reference container layer."""
