"""`skipdiff`-named drop-in: the reference package's import surface
(/root/reference/pkg/src/skipdiff/__init__.py) served by the B200 path with
host-numpy return types (paper_2603_25872_b200/numpy_api.py).  Put `dropin/`
on sys.path ahead of any real skipdiff to switch an existing caller over.
config / cli / verify (host plumbing, out of scope: DESIGN.md section 7) are not
provided."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2603_25872_b200.numpy_api import *  # noqa: E402,F401,F403
from paper_2603_25872_b200.numpy_api import __all__  # noqa: E402,F401
