"""Golden logits of the config-5 ResNet-50 program from the UNMODIFIED reference interpreter.

    python tests/golden/make_golden_resnet.py [--full]

The program text comes from paper_1903_06498_b200.workloads.resnet50 (validated clean
by the reference's validate_static); inputs are the reference's random_inputs
(tests/support.h:55-70, seed 1005), regenerated bit-identically on the GPU box by
oracle.random_inputs, so only the logits are stored.  The reduced case (32x32 image,
full widths, batch 2) runs in ~15 s; --full adds the 224x224 batch-1 network
(~4.1e9 MACs, several minutes of reference CPU time).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Ref, random_inputs  # noqa: E402
from paper_1903_06498_b200 import workloads as W  # noqa: E402

CASES = {
    "resnet50_img32_b2": dict(N=2, image=32),
    "resnet50_img224_b1": dict(N=1, image=224),
}


def make(name, N, image, seed=1005):
    text, info = W.resnet50(N, image=image)
    prog = Ref.parse(text)
    n, msg = prog.validate()
    assert n == 0, msg
    store = Ref.random_inputs(prog, seed)
    mine = random_inputs(prog.buffers(), seed)
    for k, (bits, arr) in store.items():
        if k in mine:
            assert np.array_equal(mine[k], arr), k
    t0 = time.time()
    out = Ref.execute(prog, store)
    dt = time.time() - t0
    os.makedirs(os.path.join(HERE, "resnet"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "resnet", name + ".npz"), logits=out["Logits"][1], N=N, image=image, seed=seed,
                        seconds=dt, macs=info["macs"])
    print(f"{name}: {dt:.1f} s reference time, {info['macs'] / 1e9:.3f} GMAC")


if __name__ == "__main__":
    make("resnet50_img32_b2", **CASES["resnet50_img32_b2"])
    if "--full" in sys.argv:
        make("resnet50_img224_b1", **CASES["resnet50_img224_b1"])
