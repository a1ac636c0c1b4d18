"""Exception types raised at the Python boundary of the B200 evaluator.

Mirrors the subset of the reference's ``opfkit.errors`` hierarchy
(`pkg/src/opfkit/errors.py:9-134`) that the hot path and its packer can
raise, under the same names, so callers catching ``Disconnected`` or
``DimensionMismatch`` keep working after the switch.
"""

from __future__ import annotations


class OpfkitError(Exception):
    """Root of every error raised by this package (errors.py:9)."""


class UnknownElement(OpfkitError):
    """errors.py:45."""


class UnknownOutage(UnknownElement):
    """A contingency names an element that is absent or already off (errors.py:49)."""


class IslandingDetected(OpfkitError):
    """A branch outage splits the network (errors.py:53)."""


class TargetOnNonWind(OpfkitError):
    """A scenario targets a generator that is not wind (errors.py:57)."""


class UnknownBus(OpfkitError):
    """errors.py:61."""


class IndexOutOfRange(OpfkitError):
    """errors.py:65."""


class Disconnected(OpfkitError):
    """The in-service network is not one island (errors.py:69; raised at acopf.py:97,398)."""


class EmptyScenarioSet(OpfkitError):
    """errors.py:103."""


class TopologyMismatch(OpfkitError):
    """Periods of one composite differ in topology (errors.py:121)."""


class DimensionMismatch(OpfkitError):
    """A vector has the wrong length for its layout (errors.py:125; acopf.py:470)."""


class InvalidPlan(OpfkitError):
    """errors.py:129."""


class DeviceError(OpfkitError):
    """The CUDA library reported a failure (status != 0 across the C ABI)."""
