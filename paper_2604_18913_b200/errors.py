"""Exception families of the reference (errors.py:11-56), for drop-in parity.

Contract violations on the hot path (bad ids, k < 1, max_paths < 0) raise
``ValueError`` exactly as the reference's incidence layer does; these
classes cover the partitioned layer (partition.py:68-75 raises UsageError,
engine.py:58-67 IntegrityError).
"""


class TripleHopError(Exception):
    """Base class for all package-specific errors."""


class UsageError(TripleHopError):
    """Invalid request parameters (bad partition count, rank, flags)."""


class DataError(TripleHopError):
    """Malformed input data."""


class ArchiveError(DataError):
    """Base for binary archive load failures (archive.py)."""


class BadMagicError(ArchiveError):
    """The file does not start with the LKG1 magic."""


class VersionError(ArchiveError):
    """Unsupported archive format version."""


class TruncatedError(ArchiveError):
    """The archive is shorter (or longer) than its header says."""


class ChecksumError(ArchiveError):
    """CRC32 mismatch over header + payload."""


class IntegrityError(DataError):
    """Cross-rank inconsistency (plan/world mismatch, malformed exchange)."""
