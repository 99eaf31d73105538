"""skipdiff.transitions on the B200 path (see dropin/skipdiff/__init__.py)."""

from paper_2603_25872_b200.numpy_api import *  # noqa: F401,F403
