"""Exception hierarchy of the CHR host API.

Class names, bases and attributes match the reference's error module
(isochr/errors.py) so code written against the reference -- including its
``pytest.raises(...)`` checks -- keeps working.  ``_abi.check`` maps the C-ABI
status codes (include/chr.h ``chr_status_t``) onto these classes.
"""


class IsochrError(Exception):
    """Root of every error raised by this package."""


def _simple(name: str, doc: str):
    return type(name, (IsochrError, ValueError), {"__doc__": doc})


ParameterError = _simple("ParameterError", "Invalid argument (CHR_E_PARAMETER).")
CorruptPayloadError = _simple("CorruptPayloadError", "Payload CRC or token stream invalid (CHR_E_CORRUPT).")
UnsupportedCodecError = _simple("UnsupportedCodecError", "Codec id not registered (CHR_E_UNSUPPORTED_CODEC).")
BadMagicError = _simple("BadMagicError", "File is not a CHR archive (wrong magic).")
VersionError = _simple("VersionError", "Unsupported CHR format version.")
ChecksumError = _simple("ChecksumError", "CHR file trailer CRC or table inconsistent.")


class NonFiniteSampleError(IsochrError, ValueError):
    """A NaN/Inf sample; ``index`` is its flat (x-fastest) position (CHR_E_NONFINITE)."""

    def __init__(self, index: int, value: float):
        self.index, self.value = index, value
        super().__init__(f"sample {index} is not finite ({value!r})")


class RawSizeMismatchError(IsochrError, ValueError):
    """Raw file size disagrees with dims * dtype width."""

    def __init__(self, path, expected: int, actual: int):
        self.path, self.expected, self.actual = path, expected, actual
        super().__init__(f"{path}: {actual} bytes on disk, dims/dtype need {expected}")


class NoSuchIsovalueError(IsochrError, ValueError):
    """Isovalue not stored in the archive (use snap=True for the nearest)."""

    def __init__(self, requested: float, candidates):
        self.requested, self.candidates = requested, list(candidates)
        super().__init__(f"{requested!r} not in stored candidates {self.candidates} (snap=True picks the nearest)")


class InsufficientAccuracyError(IsochrError, ValueError):
    """Request asks for more topology accuracy than the archive stores."""

    def __init__(self, requested: float, stored: float):
        self.requested, self.stored = requested, stored
        super().__init__(f"accuracy {requested} requested, archive built at {stored}")
