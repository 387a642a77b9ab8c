"""The "bgmf-b200" CLI variant (paper_2304_13724_b200.cli_plugin; the
reference's plug point is cli.py:47-51).  CPU side, in a subprocess that
imports the unmodified reference package (present in the build container,
skipped elsewhere): registration into the reference CLI's own VARIANTS table
(and its --variant choices), the field-by-field conversion of the reference's
RatingsDataset / TrainConfig / schedules, and a converted result that the
reference's own writers accept.  The GPU run through the reference CLI is
ref_suite/test_variant_plugin.py."""

import os
import subprocess
import sys
import textwrap

import pytest

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import io, sys
    sys.path.insert(0, %r)
    sys.path.insert(0, %r)
    try:
        import matplotlib  # noqa: F401
    except ImportError:  # absent in this image: the suite's placeholder stand-in
        sys.path.insert(0, %r)
    import numpy as np
    import blockmf as ref
    import blockmf.cli as cli
    from blockmf.data_io import write_trace, save_model
    import paper_2304_13724_b200 as bm
    from paper_2304_13724_b200 import cli_plugin as P

    P.register()
    assert cli.VARIANTS["bgmf-b200"] is P.train_variant
    args = cli.build_parser().parse_args(["train", "--data", "x.csv", "--variant", "bgmf-b200"])
    assert args.variant == "bgmf-b200"

    cfg = ref.TrainConfig(k=4, alpha=1e-2, outer_steps=3, grid_i=2, grid_j=3, seed=5,
                          inner_schedule=ref.ConvergeEachBlock(0.05))
    ours = P.to_config(cfg)
    assert isinstance(ours, bm.TrainConfig) and isinstance(ours.inner_schedule, bm.ConvergeEachBlock)
    assert (ours.k, ours.alpha, ours.outer_steps, ours.grid_i, ours.grid_j, ours.seed,
            ours.inner_schedule.tol) == (4, 1e-2, 3, 2, 3, 5, 0.05)
    for s in (ref.Constant(2), ref.IncreasingEvery(2, 3), ref.Decreasing(4),
              ref.AdaptiveDecreasing(3)):
        o = P.to_config(ref.TrainConfig(inner_schedule=s)).inner_schedule
        assert type(o).__name__ == type(s).__name__ and o == type(o)(*[getattr(s, f) for f in s.__dataclass_fields__])

    d = ref.RatingsDataset(3, 4, np.array([0, 1, 2]), np.array([1, 2, 3]), np.array([1.0, 2.0, 3.0]))
    od = P.to_dataset(d)
    assert isinstance(od, bm.RatingsDataset) and (od.n, od.m) == (3, 4)
    assert np.array_equal(od.values, d.values)

    # a result of this package's classes comes back as the reference's
    trace = bm.ConvergenceTrace()
    trace.append(bm.TraceStep(step=0, train_rmse=1.5, test_rmse=None, seconds=0.1,
                              inner_iters=1, capped_blocks=0))
    res = bm.TrainResult(model=bm.FactorModel(np.ones((3, 2)), np.ones((4, 2))), trace=trace,
                         stop_reason="max_steps")
    back = P.to_caller_result(res, d)
    assert type(back).__module__ == "blockmf.trainer"
    assert type(back.trace).__module__ == "blockmf.core" and back.trace.last().train_rmse == 1.5
    write_trace(back.trace, io.StringIO(), {"variant": "bgmf-b200"})
    save_model(back.model, io.StringIO())
    print("ok")
""")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_SRC, "blockmf")),
                    reason="the reference package is only in the build container")
def test_register_and_convert_with_the_reference_package():
    out = subprocess.run([sys.executable, "-c", SCRIPT % (ROOT, REF_SRC, os.path.join(ROOT, "ref_suite", "stubs"))], capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-3000:]
