"""pytest plugin (-p bgmf_alias): make `import blockmf` resolve to this repo's
drop-in, so the reference package's own unit tests run unchanged against the
B200 implementation.  Submodules the reference tests import by name map to
their counterparts here (blockmf.kernel -> .kernel, blockmf.data_io -> .data)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2304_13724_b200 as _bm  # noqa: E402
from paper_2304_13724_b200 import data as _data  # noqa: E402
from paper_2304_13724_b200 import kernel as _kernel  # noqa: E402

sys.modules["blockmf"] = _bm
sys.modules["blockmf.kernel"] = _kernel
sys.modules["blockmf.data_io"] = _data
