"""Run the reference package's own unit tests against the drop-in.

The test files are NOT part of this repository (they are the reference's
sources): `python ref_suite/run.py sync` copies them, when /root/reference is
present (the build container), into ref_suite/_ref/ -- git-ignored, but it
travels to the GPU box with the gpurun snapshot like the built .so files.
`python ref_suite/run.py [fast|exact] [pytest args]` then runs them on the GPU
with `blockmf` aliased to paper_2304_13724_b200 (bgmf_alias.py):
  exact -- BGMF_EXACT=1: every train/sweep call uses the fp64 kernels, which
           the reference's bit-identity assertions need;
  fast  -- the default fp32 engine (ordered sweep where the schedule routes
           it, chunked elsewhere).
Files: test_{kernel,partition,scheduler,trainer,metrics,baselines}.py (the
hot-path suites), test_core.py / test_data_io.py (API value types and file
formats the drop-in also provides), test_cli.py with the reference's cli.py and
report.py loaded over the drop-in (the CLI's VARIANTS plug-in path; matplotlib
is absent here, so figures are placeholder files), and conftest.py."""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/tests"
FILES = ["conftest.py", "test_kernel.py", "test_partition.py", "test_scheduler.py",
         "test_trainer.py", "test_metrics.py", "test_baselines.py", "test_core.py",
         "test_data_io.py", "test_cli.py"]
# the reference's CLI and report modules, loaded on top of the drop-in as
# blockmf.cli / blockmf.report (bgmf_alias.py): its VARIANTS table then holds
# this package's trainers
SRC = "/root/reference/pkg/src/blockmf"
SRC_FILES = ["cli.py", "report.py"]


def sync() -> None:
    dst = os.path.join(HERE, "_ref")
    os.makedirs(dst, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(REF, f), os.path.join(dst, f))
    for f in SRC_FILES:
        shutil.copyfile(os.path.join(SRC, f), os.path.join(dst, f))
    print(f"copied {len(FILES) + len(SRC_FILES)} files from {REF}, {SRC} to {dst}")


def run(mode: str, extra: list[str]) -> int:
    env = dict(os.environ)
    env["PYTHONPATH"] = HERE + os.pathsep + env.get("PYTHONPATH", "")
    if mode == "exact":
        env["BGMF_EXACT"] = "1"
    # explicit test files / node ids narrow the run; else the whole suite
    picked = [a for a in extra if a.endswith(".py") or "::" in a]
    # plus this repository's own test of the "bgmf-b200" CLI variant
    # (test_variant_plugin.py), which needs the reference CLI copied by sync
    ours = [os.path.join(HERE, "test_variant_plugin.py")] \
        if os.path.exists(os.path.join(HERE, "_ref", "cli.py")) else []
    cmd = [sys.executable, "-m", "pytest", "-p", "bgmf_alias", "-q", "-rf",
           "-p", "no:cacheprovider", "--rootdir", os.path.join(HERE, "_ref"),
           *([] if picked else [os.path.join(HERE, "_ref"), *ours]), *extra]
    return subprocess.call(cmd, env=env, cwd=os.path.join(HERE, "_ref"))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "exact"
    if what == "sync":
        sync()
    else:
        sys.exit(run(what, sys.argv[2:]))
