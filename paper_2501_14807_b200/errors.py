"""Exception classes of the drop-in surface.

The reference gives every error a stable wire ``code`` (reference ``errors.py:1-97``); the names,
codes and the one inheritance edge (``UVRangeError`` is a ``ParseError``, ``errors.py:12``) are
part of the API a caller can observe, so they are reproduced exactly -- from the table below
rather than as 24 hand-written class bodies.
"""


class MeshLayersError(Exception):
    """Root of the hierarchy (reference errors.py:4)."""
    code = "error"


# (class name, wire code, base class name) -- reference errors.py:8-97
_TABLE = (
    ("ParseError", "parse_error", "MeshLayersError"),
    ("UVRangeError", "uv_range", "ParseError"),
    ("MissingUVs", "missing_uvs", "MeshLayersError"),
    ("EmptyMesh", "empty_mesh", "MeshLayersError"),
    ("DegenerateCamera", "degenerate_camera", "MeshLayersError"),
    ("CapacityExceeded", "capacity_exceeded", "MeshLayersError"),
    ("TargetMismatch", "target_mismatch", "MeshLayersError"),
    ("BadPalette", "bad_palette", "MeshLayersError"),
    ("UnknownTable", "unknown_table", "MeshLayersError"),
    ("BadMagic", "bad_magic", "MeshLayersError"),
    ("UnsupportedVersion", "unsupported_version", "MeshLayersError"),
    ("TruncatedStream", "truncated_stream", "MeshLayersError"),
    ("ChecksumMismatch", "checksum_mismatch", "MeshLayersError"),
    ("StaleDepth", "stale_depth", "MeshLayersError"),
    ("LayerMeshMismatch", "layer_mesh_mismatch", "MeshLayersError"),
    ("MemoryBudgetExceeded", "memory_budget_exceeded", "MeshLayersError"),
    ("DuplicateTable", "duplicate_table", "MeshLayersError"),
    ("BadSchema", "bad_schema", "MeshLayersError"),
    ("SchemaViolation", "schema_violation", "MeshLayersError"),
    ("ReservedKey", "reserved_key", "MeshLayersError"),
    ("UnknownLayer", "unknown_layer", "MeshLayersError"),
    ("BindFailure", "bind_failure", "MeshLayersError"),
    ("BadRequest", "bad_request", "MeshLayersError"),
)

__all__ = ["MeshLayersError", "BackendUnavailable"]
for _name, _code, _base in _TABLE:
    globals()[_name] = type(_name, (globals()[_base],), {"code": _code, "__module__": __name__})
    __all__.append(_name)


class BackendUnavailable(MeshLayersError):
    """Extension of this package: the CUDA library or a CUDA device is missing.  There is no
    CPU fallback -- every operation fails loudly with this error instead."""
    code = "backend_unavailable"
