"""The drop-in boundary exercised from the reference's side: oracle/_ref/dropin_test is
built from the UNMODIFIED reference sources plus include/stripe_b200_binding.hpp and runs
stripe::execute and stripe::b200::execute (the C ABI) on the same random inputs
(tests/support.h:55-70), comparing every buffer and every error code."""
import os
import subprocess

import pytest

from harness import HERE, corpus, gpu_available

BIN = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "dropin_test")


@pytest.mark.gpu
def test_reference_side_dropin(tmp_path):
    if not gpu_available():
        pytest.skip("no B200")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    from paper_1903_06498_b200 import workloads as W
    files = []
    for c in corpus():
        p = tmp_path / f"{c.name}.stripe"
        p.write_text(c.text)
        files.append(str(p))
    extra = {"c2_small": W.conv2d(2, 12, 12, 64, 64), "igemm_s2": W.conv2d(1, 9, 9, 64, 128, pad=1, stride=2),
             "fused": W.conv_fused(1, 8, 8, 64, 64), "pool": W.pool2d(2, 9, 9, 16),
             "limb": W.matmul(64, 48, 32, in_dtype="i32", out_dtype="i32"),
             "resnet_tiny": W.resnet50(1, image=32, width=8, stages=(1, 1, 1, 1), classes=10)[0]}
    for name, text in extra.items():
        p = tmp_path / f"{name}.stripe"
        p.write_text(text)
        files.append(str(p))
    r = subprocess.run([BIN, "--seed", "1001"] + files, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l]
    bad = [l for l in lines if not l.startswith(("OK", "SKIP"))]
    assert r.returncode == 0 and not bad, "\n".join(bad[:20]) + r.stderr[-2000:]
    assert sum(l.startswith("OK") for l in lines) >= len(files) - 2


@pytest.mark.gpu
def test_reference_side_dropin_concurrent_threads(tmp_path):
    """8 host threads call stripe::b200::execute at once on disjoint stores (SPEC.md:263:
    execute is reentrant); every thread's store must equal stripe::execute's."""
    if not gpu_available():
        pytest.skip("no B200")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    from paper_1903_06498_b200 import workloads as W
    progs = {"c2_small": W.conv2d(2, 12, 12, 64, 64), "igemm_s2": W.conv2d(1, 9, 9, 64, 128, pad=1, stride=2),
             "fused": W.conv_fused(1, 8, 8, 64, 64), "pool": W.pool2d(2, 9, 9, 16),
             "limb": W.matmul(64, 48, 32, in_dtype="i32", out_dtype="i32")}
    for c in corpus():
        if c.name in ("fx_matmul64", "fx_conv_relu", "fx_gather", "rnd_prog_03", "tile_conv_x3y4"):
            progs[c.name] = c.text
    files = []
    for name, text in progs.items():
        p = tmp_path / f"{name}.stripe"
        p.write_text(text)
        files.append(str(p))
    r = subprocess.run([BIN, "--seed", "77", "--threads", "8"] + files, capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if "threads=" in l]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert len(lines) >= len(files) - 1 and all(l.startswith("OK") for l in lines), r.stdout


@pytest.mark.gpu
def test_reference_side_autotile(tmp_path):
    """stripe::b200::autotile (device line counts + the reference's tile_rewrite) against
    stripe::autotile on block 0 of small programs, divisor and power-of-two spaces: same chosen
    shape, report, candidate counts, rewritten block text and exception codes (tile.cpp:475-535)."""
    if not gpu_available():
        pytest.skip("no B200")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    from paper_1903_06498_b200 import workloads as W
    progs = {"mm": W.matmul(16, 12, 20), "conv": W.conv2d(1, 8, 8, 4, 4), "pool": W.pool2d(2, 9, 9, 4)}
    for c in corpus():
        if c.name.startswith(("fx_", "rnd_text_0", "gen_", "tile_")) and c.name not in ("fx_place2",):
            progs[c.name] = c.text
    files = []
    for name, text in progs.items():
        p = tmp_path / f"{name}.stripe"
        p.write_text(text)
        files.append(str(p))
    r = subprocess.run([BIN, "--seed", "5", "--autotile", "8:512"] + files, capture_output=True, text=True,
                       timeout=900)
    lines = [l for l in r.stdout.splitlines() if " autotile " in l]
    assert r.returncode == 0, "\n".join(l for l in r.stdout.splitlines() if not l.startswith("OK"))[-3000:]
    assert len(lines) >= 2 * (len(files) - 6) and all(l.startswith("OK") for l in lines), r.stdout[-3000:]
