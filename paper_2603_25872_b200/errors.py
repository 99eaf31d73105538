"""Exception hierarchy of the drop-in.

Same class names and the same single base as skipdiff errors.py, so call
sites written against the reference (`except InvalidPlanParams`) port
unchanged.  libdrs.so status codes (include/drs.h) are mapped onto these by
_lib.check().  Classes are generated from one table: (name, reference line,
meaning).
"""


class SkipDiffError(Exception):
    """Base class of every error raised by the package (skipdiff errors.py:4)."""


_TABLE = (
    ("InvalidScheduleParams", 8, "schedule construction parameters out of range"),
    ("TimestepOutOfRange", 12, "timestep outside the schedule's 0..T range"),
    ("DimensionMismatch", 16, "state vectors of incompatible dimensions"),
    ("NonPositiveSigma", 20, "velocity oracle queried at sigma <= 0"),
    ("InvalidSkip", 24, "skip length k < 1"),
    ("VarianceTooLarge", 28, "transition variance above 1 - alpha_bar[t-k]"),
    ("IndexOutOfRange", 32, "sigma-grid index outside 0..N"),
    ("InvalidSubsequence", 36, "DDIM subsequence not strictly decreasing to 0"),
    ("InvalidPlanParams", 40, "T < 1, devices < 1, or an oversubscribed round"),
    ("PlanMismatch", 44, "executed trajectory disagrees with its block plan"),
    ("WorkerFailure", 48, "an evaluation task failed; chains the first error"),
    ("TimestepMismatch", 52, "trajectories compared over different timesteps"),
    ("EmptySet", 56, "metric called on an empty sample set"),
    ("InsufficientSamples", 60, "unbiased MMD needs >= 2 samples per set"),
    ("ParseError", 64, "malformed CSV input"),
    ("ConfigError", 68, "malformed run configuration"),
    ("SuiteNotFound", 72, "unknown verification suite"),
)

for _name, _line, _doc in _TABLE:
    globals()[_name] = type(_name, (SkipDiffError,), {
        "__doc__": f"{_doc[0].upper()}{_doc[1:]} (skipdiff errors.py:{_line}).",
        "__module__": __name__,
    })

__all__ = ["SkipDiffError"] + [n for n, _, _ in _TABLE]
