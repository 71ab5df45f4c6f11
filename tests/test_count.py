"""count_valid_points (tile.cpp:338-370) on the device, closed form per
innermost row, against the reference's tile_cost(...).useful_ops and the configs' counts."""
import pytest

from harness import corpus, gpu_available
from oracle import Ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not gpu_available():
        pytest.skip("no B200")


def test_count_matches_reference_on_corpus_blocks():
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    texts = {c.name: c.text for c in corpus() if "block [" in c.text}
    texts["conv_pad"] = W.conv2d(2, 9, 7, 4, 4)
    texts["conv_s2"] = W.conv2d(1, 11, 10, 4, 4, R=5, S=3, pad=2, stride=2)
    texts["pool"] = W.pool2d(2, 9, 9, 4)
    checked = 0
    for name, text in texts.items():
        prog = sb.parse_program(text)
        for path in ("0", "0.0"):
            try:
                exp = Ref.useful_ops(text, path)
            except Exception:
                continue  # no block there, or aliases (the reference refuses those too)
            assert prog.count_valid_points(path) == exp, (name, path)
            checked += 1
    assert checked >= 20


def test_count_config_scale():
    """C2 (3.6118e9 useful MACs) and C5's stem, in milliseconds instead of
    the reference's minutes."""
    import paper_1903_06498_b200 as sb
    from paper_1903_06498_b200 import workloads as W
    p = sb.parse_program(W.conv2d(32, 56, 56, 64, 64))
    assert p.count_valid_points("0") == W.conv_useful_macs(32, 56, 56, 64, 64) == 3611820032
    stem = sb.parse_program(W.conv2d(128, 224, 224, 3, 64, R=7, S=7, pad=3, stride=2))
    # 7x7/2 pad 3 on 224: per axis sum over outputs of in-bounds taps
    ax = sum(1 for x in range(112) for i in range(7) if 0 <= 2 * x + i - 3 < 224)
    assert stem.count_valid_points("0") == 128 * ax * ax * 3 * 64
