"""Exception taxonomy of the reference (errors.py:4-61), re-raised by the
Python surface when the C-ABI reports a status or a per-env flag.

The device path never raises mid-step: kernels write per-env masks
(nonfinite, spawn failure) and the host maps them to these types at the next
synchronisation point.
"""


class QuadsimError(Exception):
    """Root of every error raised by this package."""


class NonFiniteState(QuadsimError):
    """Some agents' states left the finite range (errors.py:8-19)."""

    def __init__(self, state, mask):
        self.state, self.mask = state, mask
        try:
            bad = [int(i) for i in mask.nonzero()[0]]
        except Exception:  # torch masks
            bad = mask.nonzero().flatten().tolist()
        super().__init__(f"non-finite state components for agents {bad}")


class EmptyScene(QuadsimError):
    pass


class ParseError(QuadsimError):
    def __init__(self, message, path=None, line=None):
        self.path, self.line = path, line
        where = "".join(x for x in (str(path) if path is not None else "", f":{line}" if line is not None else ""))
        super().__init__(f"{where}: {message}" if where else message)


class ConfigError(QuadsimError):
    pass


class SpawnFailure(QuadsimError):
    pass


class NotReset(QuadsimError):
    pass


class ActionShapeMismatch(QuadsimError):
    pass


class InvalidNoiseForSensor(QuadsimError):
    pass


class DegenerateAttitude(QuadsimError):
    pass


class NativeError(QuadsimError):
    """The sm_100a library returned a non-zero status (qb_last_error())."""


class InvalidNoiseForSensor(QuadsimError):
    """Noise kind is not defined for the given sensor data type (errors.py:56-57)."""
