"""Shared helpers for the parity tests: golden corpus, oracle and device runners."""
import glob
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


class Case:
    def __init__(self, path):
        z = np.load(path)
        self.name = os.path.basename(path)[:-4]
        self.text = str(z["text"])
        self.error = str(z["error"])
        self.note = str(z["note"])
        self.inputs = {}
        self.expected = {}
        for k in z.files:
            if k.startswith("in_"):
                n = k[3:]
                self.inputs[n] = (int(z["bits_" + n]), z[k].astype(np.int64))
            elif k.startswith("out_"):
                self.expected[k[4:]] = z[k].astype(np.int64)

    def __repr__(self):
        return self.name


def corpus():
    return [Case(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))]


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False


def run_device(text, inputs, disable_tc=False, order=0):
    """Runs the B200 executor on int64-carrier inputs; returns dict name -> int64 array."""
    import paper_1903_06498_b200 as sb
    prog = sb.parse_program(text)
    store = {n: sb.Buffer(bits, arr.copy()) for n, (bits, arr) in inputs.items()}
    sb.prepare_outputs(prog, store)
    sb.execute(prog, store, sb.ExecOptions(order=sb.IterOrder(order), disable_tensor_cores=disable_tc))
    return {n: b.data for n, b in store.items()}
