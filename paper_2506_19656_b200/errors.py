"""Exception hierarchy of the drop-in.

When the reference package is importable its own classes are re-exported, so
``except cubevid.errors.ConfigurationError`` in existing callers catches what
this path raises without any aliasing; otherwise the same names and nesting
are defined here (/root/reference/pkg/src/cubevid/errors.py:4-21).
"""

try:  # the reference's own classes, when it is installed next to this package
    from cubevid.errors import (CodecError, ConfigurationError, CorruptStreamError,  # noqa: F401
                                CubevidError, ManifestError)

    SHARED_WITH_REFERENCE = True
except ImportError:
    SHARED_WITH_REFERENCE = False

    class CubevidError(Exception):
        """Base class for all errors raised by the B200 path."""

    class ConfigurationError(CubevidError):
        """Invalid bit depth, range, shape or non-finite data (reference convention)."""

    class CodecError(CubevidError):
        """The external encoder or decoder failed (raised by codec plug-ins)."""

    class CorruptStreamError(CodecError):
        """Frame buffers whose size is not a whole number of frames."""

    class ManifestError(CubevidError):
        """A container directory is missing files or carries a bad manifest."""
