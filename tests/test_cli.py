"""`stripec run` / `stripec diff` on the B200 (paper_1903_06498_b200/
stripec_b200, a pure C-ABI client) with the reference's native-width buffer directories
(io.cpp:28-85).  Expected values come from the unmodified reference interpreter."""
import os
import subprocess

import numpy as np
import pytest

from harness import GOLDEN, HERE, corpus, gpu_available

BIN = os.path.join(os.path.dirname(HERE), "paper_1903_06498_b200", "stripec_b200")
NP = {8: np.int8, 16: np.int16, 32: np.int32}
NAME = {8: "i8", 16: "i16", 32: "i32"}


def write_dir(path, inputs):
    os.makedirs(path, exist_ok=True)
    with open(os.path.join(path, "buffers.txt"), "w") as f:
        for n, (bits, a) in inputs.items():
            f.write(f"{n} {NAME[bits]} {a.size}\n")
            a.astype(NP[bits]).tofile(os.path.join(path, f"{n}.bin"))


def read_dir(path):
    out = {}
    for line in open(os.path.join(path, "buffers.txt")):
        n, dt, cnt = line.split()
        bits = {"i8": 8, "i16": 16, "i32": 32}[dt]
        out[n] = np.fromfile(os.path.join(path, f"{n}.bin"), dtype=NP[bits]).astype(np.int64)
        assert out[n].size == int(cnt)
    return out


def cli(*args):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=300)


def test_cli_parse_round_trip(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("stripec_b200 not built")
    c = [c for c in corpus() if c.name == "fx_conv_relu"][0]
    p = tmp_path / "p.stripe"
    p.write_text(c.text)
    r = cli("parse", str(p))
    assert r.returncode == 0 and r.stdout == c.text


def test_cli_usage_and_parse_errors(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("stripec_b200 not built")
    assert cli("run").returncode == 2
    p = tmp_path / "bad.stripe"
    p.write_text("block [x:2]:2 ( ) { 0: $a = frobnicate() }")
    r = cli("run", str(p), "--data", str(tmp_path))
    assert r.returncode == 1 and r.stderr.startswith("error ")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["fx_matmul64", "fx_conv_relu", "fx_maxpool", "gen_conv_10x12x16x32_i8",
                                  "fx_fig6a_fixed_i32"])
def test_cli_run_matches_reference(tmp_path, name):
    if not gpu_available():
        pytest.skip("no B200")
    c = [c for c in corpus() if c.name == name][0]
    prog = tmp_path / "p.stripe"
    prog.write_text(c.text)
    write_dir(tmp_path / "in", c.inputs)
    r = cli("run", str(prog), "--data", str(tmp_path / "in"), "--out", str(tmp_path / "out"))
    assert r.returncode == 0, r.stderr
    got = read_dir(tmp_path / "out")
    for n, exp in c.expected.items():
        if n in got:
            np.testing.assert_array_equal(got[n], exp, err_msg=n)
    r = cli("run", str(prog), "--data", str(tmp_path / "in"))
    for line in r.stdout.splitlines():
        n, dt, cnt, s = line.split()
        assert int(s.split("=")[1]) == int(c.expected[n].sum()), line


@pytest.mark.gpu
def test_cli_diff(tmp_path):
    """acceptance.cpp:267-316: fig6a_fixed_i32 and fig6b_i32 agree on random inputs; a
    different program reports its first differing element."""
    if not gpu_available():
        pytest.skip("no B200")
    by = {c.name: c for c in corpus()}
    a, b = by["fx_fig6a_fixed_i32"], by["fx_fig6b_i32"]
    (tmp_path / "a.stripe").write_text(a.text)
    (tmp_path / "b.stripe").write_text(b.text)
    write_dir(tmp_path / "in", a.inputs)
    r = cli("diff", str(tmp_path / "a.stripe"), str(tmp_path / "b.stripe"), "--data", str(tmp_path / "in"))
    assert r.returncode == 0 and r.stdout.strip() == "identical", r.stdout + r.stderr
    (tmp_path / "c.stripe").write_text(a.text.replace("$O = mul(", "$O = add(").replace("= mul(", "= add(", 1))
    r = cli("diff", str(tmp_path / "a.stripe"), str(tmp_path / "c.stripe"), "--data", str(tmp_path / "in"))
    if "add(" in (tmp_path / "c.stripe").read_text() and (tmp_path / "c.stripe").read_text() != a.text:
        assert r.returncode == 1 and "a=" in r.stdout and "b=" in r.stdout, r.stdout + r.stderr
