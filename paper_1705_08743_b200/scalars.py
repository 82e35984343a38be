"""Scalar definitions of the two path semirings (pkg/src/semimat/scalars.py).

These are the per-cell rules the device kernels implement lane-wise; they are
kept as plain Python so user code that imported them from the reference keeps
working.  S = 2**width - 1 is the saturation limit (scalars.py:16-23).
"""

SAT_WIDTHS = (8, 16, 32)


def sat_limit(width: int) -> int:
    """S = 2**width - 1 for width in (8, 16, 32) (scalars.py:19-23)."""
    if width not in SAT_WIDTHS:
        raise ValueError(f"unsupported width {width}, expected one of {SAT_WIDTHS}")
    return (1 << width) - 1


def bool_add(a: int, b: int) -> int:
    """Boolean (+): the larger bit (scalars.py:26-28)."""
    return max(a, b)


def bool_mul(a: int, b: int) -> int:
    """Boolean (x): the smaller bit (scalars.py:31-33)."""
    return min(a, b)


def sat_mul(a: int, b: int, width: int = 8) -> int:
    """Anti-distance (x): max(a + b - S, 0) (scalars.py:36-43)."""
    return max(a + b - sat_limit(width), 0)


def sat_neg(a: int, width: int = 8) -> int:
    """Complement at width, S - a (scalars.py:46-52)."""
    return sat_limit(width) - a


def delta(a: int, width: int = 8) -> int:
    """Distance encoded by anti-distance value a (scalars.py:55-57)."""
    return sat_limit(width) - a


def dist_mul(a: int, b: int, width: int = 8) -> int:
    """Distance (x): min(a + b, S) (scalars.py:60-68)."""
    return min(a + b, sat_limit(width))
