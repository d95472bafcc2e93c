"""Error classes of the section-graph executor.

Same class names, base class and ``(message, **context)`` convention as the
reference hierarchy (``/root/reference/pkg/src/maestro/errors.py:10-134``), so
code written against the reference catches the same exceptions.  Device
kernels cannot raise: they set a device error word ``(code, sample, aux)``
that the host shim (:mod:`._native`) decodes into one of these classes via
:data:`DEVICE_CODES`.
"""

from __future__ import annotations


class MaestroError(Exception):
    """Root of every error raised by this package (errors.py:10-22)."""

    def __init__(self, message: str, **context: object):
        super().__init__(message)
        # None-valued context entries are dropped, as in the reference.
        self.context = {key: val for key, val in context.items() if val is not None}

    def __str__(self) -> str:
        text = super().__str__()
        if not self.context:
            return text
        detail = ", ".join(f"{key}={self.context[key]}" for key in sorted(self.context))
        return f"{text} ({detail})"


def _leaf(name: str, doc: str = "") -> type:
    return type(name, (MaestroError,), {"__doc__": doc or name, "__module__": __name__})


# graph construction / spec (errors.py:25-75)
ParseError = _leaf("ParseError", "Workload spec could not be parsed.")
DuplicateSection = _leaf("DuplicateSection")
NoCriticalSection = _leaf("NoCriticalSection")
MultipleCriticalSections = _leaf("MultipleCriticalSections")
CycleDetected = _leaf("CycleDetected")
UnknownSection = _leaf("UnknownSection")
DisconnectedAuxiliary = _leaf("DisconnectedAuxiliary", "Auxiliary lies on no path through the critical section.")
EdgeNotFound = _leaf("EdgeNotFound")
InvalidDims = _leaf("InvalidDims")
BothActivated = _leaf("BothActivated", "Sample activates two submodules merged into one section.")
ActivationError = _leaf("ActivationError", "Activated-section set inconsistent with the timing.")
NegativeTime = _leaf("NegativeTime")
EmptyBatch = _leaf("EmptyBatch")

# cost model / planning (errors.py:78-101)
InvalidConfig = _leaf("InvalidConfig", "Parallel degrees do not divide the structural parameters.")
NoFeasibleConfig = _leaf("NoFeasibleConfig")
CannotAvoidStall = _leaf("CannotAvoidStall")
FanoutViolation = _leaf("FanoutViolation", "DP^aux x fanout != DP^neighbor on some edge.")
InfeasiblePlan = _leaf("InfeasiblePlan")

# scheduler / executor (errors.py:106-115)
FanoutMismatch = _leaf("FanoutMismatch")
InconsistentSchedule = _leaf("InconsistentSchedule")
DependencyDeadlock = _leaf("DependencyDeadlock")

# handoff / reshard (errors.py:121-134)
IncompatibleShapes = _leaf("IncompatibleShapes")
ChannelClosed = _leaf("ChannelClosed")
SlotExhausted = _leaf("SlotExhausted", "Destination slot budget exceeded (backpressure, never a drop).")
FragmentTimeout = _leaf("FragmentTimeout")

# Not in the reference: the native library itself failed (missing .so, CUDA
# error).  Never used to signal a domain error.
NativeError = _leaf("NativeError", "CUDA extension missing or a CUDA call failed.")

# Device error word codes -> class.  Must match include/maestro_b200.h.
DEVICE_CODES = {
    1: NegativeTime,
    2: BothActivated,
    3: ActivationError,
    4: InvalidDims,
    5: FanoutMismatch,
    6: EmptyBatch,
    7: InconsistentSchedule,
    8: FanoutViolation,
}
