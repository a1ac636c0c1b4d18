"""Exception types raised at the Python boundary of the B200 evaluator.

Mirrors the subset of the reference's ``opfkit.errors`` hierarchy
(`pkg/src/opfkit/errors.py:9-134`) that the hot path and its packer can
raise, under the same names, so callers catching ``Disconnected`` or
``DimensionMismatch`` keep working after the switch.  When the reference
itself is importable (``opfkit`` installed beside this package), every class
also derives from the same-named ``opfkit.errors`` class, so
``except opfkit.errors.Disconnected`` catches this package's errors too.
"""

from __future__ import annotations

try:             # optional: the reference installed beside this package (drop-in interop)
    import opfkit.errors as _ref
except Exception:           # noqa: BLE001 -- absent on GPU boxes and in plain installs
    _ref = None


def _with_ref(name: str, *own):
    """Bases of error ``name``: this package's parent, plus the reference's same-named class
    when opfkit is importable, so ``except opfkit.errors.X`` also catches this package's X."""
    r = getattr(_ref, name, None) if _ref is not None else None
    if isinstance(r, type) and issubclass(r, BaseException):
        return (*own, r) if own and own[0] is not Exception else (r,)
    return own


class OpfkitError(*_with_ref("OpfkitError", Exception)):
    """Root of every error raised by this package (errors.py:9)."""


class UnknownElement(*_with_ref("UnknownElement", OpfkitError)):
    """errors.py:45."""


class UnknownOutage(*_with_ref("UnknownOutage", UnknownElement)):
    """A contingency names an element that is absent or already off (errors.py:49)."""


class IslandingDetected(*_with_ref("IslandingDetected", OpfkitError)):
    """A branch outage splits the network (errors.py:53)."""


class TargetOnNonWind(*_with_ref("TargetOnNonWind", OpfkitError)):
    """A scenario targets a generator that is not wind (errors.py:57)."""


class UnknownBus(*_with_ref("UnknownBus", OpfkitError)):
    """errors.py:61."""


class IndexOutOfRange(*_with_ref("IndexOutOfRange", OpfkitError)):
    """errors.py:65."""


class Disconnected(*_with_ref("Disconnected", OpfkitError)):
    """The in-service network is not one island (errors.py:69; raised at acopf.py:97,398)."""


class EmptyScenarioSet(*_with_ref("EmptyScenarioSet", OpfkitError)):
    """errors.py:103."""


class TopologyMismatch(*_with_ref("TopologyMismatch", OpfkitError)):
    """Periods of one composite differ in topology (errors.py:121)."""


class DimensionMismatch(*_with_ref("DimensionMismatch", OpfkitError)):
    """A vector has the wrong length for its layout (errors.py:125; acopf.py:470)."""


class InvalidPlan(*_with_ref("InvalidPlan", OpfkitError)):
    """errors.py:129."""


class DeviceError(*_with_ref("DeviceError", OpfkitError)):
    """The CUDA library reported a failure (status != 0 across the C ABI)."""
