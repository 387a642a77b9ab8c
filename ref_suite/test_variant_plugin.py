"""(This repository's test, not a reference file.)  The reference CLI -- its own
cli.py, loaded over the drop-in by bgmf_alias -- with "bgmf-b200" added to its
VARIANTS table by paper_2304_13724_b200.cli_plugin.register (the plug point of
cli.py:47-51): `train --variant bgmf-b200` runs on the GPU, writes the
reference's trace and model files, and matches `--variant bgmf` (the same
engine) bit for bit with timing off; `evaluate` reads the model back."""

import blockmf.cli as cli
from blockmf.data_io import read_trace
from paper_2304_13724_b200 import cli_plugin


def run(*argv):
    return cli.main([str(a) for a in argv])


def test_train_variant_bgmf_b200(tmp_path, capsys):
    cli_plugin.register(cli.VARIANTS)
    data = tmp_path / "d.csv"
    assert run("gen", "--out", data, "--n", 40, "--m", 30, "--low", 1, "--high", 9,
               "--seed", 4) == cli.EXIT_OK
    outs = {}
    for variant in ("bgmf-b200", "bgmf"):
        trace, model = tmp_path / f"{variant}.csv", tmp_path / f"{variant}.txt"
        assert run("train", "--data", data, "--variant", variant, "--grid", "2x3", "--k", 4,
                   "--alpha", 1e-2, "--outer-steps", 5, "--no-timing", "--no-early-stop",
                   "--no-plot", "--trace", trace, "--model-out", model) == cli.EXIT_OK
        outs[variant] = (trace.read_text(), model.read_text())
    printed = capsys.readouterr().out
    assert "bgmf-b200: 5 steps, stop=max_steps" in printed
    # same engine behind both names: the files differ only in the recorded variant name
    t_new, m_new = outs["bgmf-b200"]
    t_old, m_old = outs["bgmf"]
    assert m_new == m_old
    assert t_new.replace("bgmf-b200", "bgmf") == t_old
    config, trace = read_trace(str(tmp_path / "bgmf-b200.csv"))
    assert config["variant"] == "bgmf-b200" and len(trace) == 5
    assert run("evaluate", "--model", tmp_path / "bgmf-b200.txt", "--data", data) == cli.EXIT_OK
