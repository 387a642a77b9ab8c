"""pytest plugin (-p bgmf_alias): make `import blockmf` resolve to this repo's
drop-in, so the reference package's own unit tests run unchanged against the
B200 implementation.  Submodules the reference tests import by name map to
their counterparts here (blockmf.kernel -> .kernel, blockmf.data_io -> .data).
When `run.py sync` has copied the reference's cli.py / report.py into _ref/,
they are loaded as blockmf.cli / blockmf.report on top of the drop-in: the
reference's own CLI (its VARIANTS table, cli.py:47-51) then drives this
package's GPU trainers -- the plug-in path of SURVEY 8(f)-2, exercised by the
reference's test_cli.py."""

import importlib
import importlib.util
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
for _name in ("core", "baselines", "metrics", "scheduler", "trainer", "partition"):
    sys.modules["blockmf." + _name] = importlib.import_module("paper_2304_13724_b200." + _name)

_REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")
try:
    import matplotlib  # noqa: F401
except ImportError:  # not in this image: a placeholder-writing stand-in
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "stubs"))
for _name in ("report", "cli"):
    _path = os.path.join(_REF, _name + ".py")
    if os.path.exists(_path):
        _spec = importlib.util.spec_from_file_location("blockmf." + _name, _path)
        _mod = importlib.util.module_from_spec(_spec)
        _mod.__package__ = "blockmf"
        sys.modules["blockmf." + _name] = _mod
        _spec.loader.exec_module(_mod)
        setattr(_bm, _name, _mod)
