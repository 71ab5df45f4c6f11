"""Exact integer restatement of conv / fused-epilogue / ResNet programs in PyTorch (test-side
checker for shapes the CPU oracles cannot finish quickly).

Semantics follow the reference interpreter: int64 temps, values wrapped only at store
(apply_aggregation, ir.cpp:79-97; wrap_value, ir.cpp:39-48), add-aggregation wraps
modulo the buffer width, locals start at zero (interp.cpp:433-453).  Convolutions are
evaluated in float64, which is exact while |sum| < 2^53 (i8 x i8 products, <= 2^20 terms).
The restatement is pinned against the reference oracle on the reduced variants in
tests/test_gpu_igemm.py / test_resnet.py.
"""
import numpy as np


def wrap(bits, x):
    import torch
    m = 1 << bits
    x = torch.remainder(x + (m >> 1), m) - (m >> 1)
    return x


def conv_exact(x_nhwc, w_rskc, stride, pad, device):
    """sum_{i,j,c} x[n, s*p+i-pad, s*q+j-pad, c] * w[i, j, k, c] as int64 (zero padding)."""
    import torch
    x = torch.as_tensor(np.asarray(x_nhwc), device=device).permute(0, 3, 1, 2).double()
    w = torch.as_tensor(np.asarray(w_rskc), device=device).permute(2, 3, 0, 1).double()
    o = torch.nn.functional.conv2d(x, w, stride=stride, padding=pad)
    return o.permute(0, 2, 3, 1).round().long()


def conv_layer_exact(x, w, b, stride, pad, relu=True, residual=None, out_bits=8, device="cuda", lo=0):
    """conv_layer semantics: T = wrap32(conv); out = wrap_out(max(T + b (+ res), 0))."""
    import torch
    t = wrap(32, conv_exact(x, w, stride, pad, device))
    s = t + torch.as_tensor(np.asarray(b), device=device).long()
    if residual is not None:
        s = s + residual.long()
    if relu:
        s = torch.clamp(s, min=lo)
    return wrap(out_bits, s)


def resnet_exact(info, inputs, image, width, stages, classes, device="cuda"):
    """Logits of workloads.resnet50 with the given int64 input carriers (dict name -> array)."""
    import torch
    convs = info["convs"]
    N = None

    def arr(name, shape):
        return np.asarray(inputs[name]).reshape(shape)

    ci = [0]

    def conv(x, relu=True, residual=None):
        c = convs[ci[0]]
        l = ci[0]
        ci[0] += 1
        w = arr(f"W{l}", (c["R"], c["S"], c["K"], c["C"]))
        b = arr(f"B{l}", (c["K"],))
        xin = x.cpu().numpy() if hasattr(x, "cpu") else x
        return conv_layer_exact(xin, w, b, c["stride"], c["pad"], relu, residual, 8, device)

    X = np.asarray(inputs["X"])
    N = X.size // (image * image * convs[0]["C"])
    a = conv(X.reshape(N, image, image, convs[0]["C"]))
    # 3x3/2 max-pool, pad 1, into a zero-initialised local
    t = a.permute(0, 3, 1, 2).double()
    pooled = torch.nn.functional.max_pool2d(t, 3, 2, 1)  # -inf padding == skipped taps
    a = torch.clamp(pooled, min=0).permute(0, 2, 3, 1).long()
    for si, nb in enumerate(stages):
        for bi in range(nb):
            if bi == 0:
                sc = conv(a, relu=False)
            else:
                sc = a
            t1 = conv(a)
            t2 = conv(t1)
            a = conv(t2, relu=True, residual=sc)
    g = wrap(8, a.sum(dim=(1, 2)))  # [N, C]
    C = g.shape[1]
    wfc = torch.as_tensor(arr("Wfc", (classes, C)), device=device).double()
    t = wrap(32, (g.double() @ wfc.t()).round().long())
    return wrap(32, t + torch.as_tensor(arr("Bfc", (classes,)), device=device).long()).cpu().numpy()
