"""Stripe program builders for the BASELINE.json configurations.

Shapes follow the reference generators (proj/tests/support.cpp:50-155:
gen_matmul / gen_conv / gen_maxpool) extended with a batch index, NHWC layout
and configurable dtypes, exactly as SURVEY §8(d) specifies the configs:

  C2  conv2d 3x3 NHWC 56x56x64->64, batch 32, halo constraints
  C4a 2x2 max-pool 112x112x64, batch 128
  C4b global sum 7x7x2048, batch 1024

All return canonical .stripe text that both the reference parser and ours accept
(for integer dtypes).
"""


def conv2d(N, H, W, C, K, R=3, S=3, in_dtype="i8", out_dtype="i32", pad=1, stride=1):
    """O[n,x,y,k] += I[n, s*x+i-pad, s*y+j-pad, c] * F[i,j,k,c], constraints keep taps in bounds."""
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    sI = (H * W * C, W * C, C, 1)
    sF = (S * K * C, K * C, C, 1)
    sO = (P * Q * K, Q * K, K, 1)
    pts = N * P * Q * R * S * C * K
    cons = []
    if pad:
        cons = [f"{_aff((stride, 'x'), (1, 'i'), -pad)} >= 0", f"{_aff((-stride, 'x'), (-1, 'i'), H - 1 + pad)} >= 0",
                f"{_aff((stride, 'y'), (1, 'j'), -pad)} >= 0", f"{_aff((-stride, 'y'), (-1, 'j'), W - 1 + pad)} >= 0"]
    lines = "\n".join("\t\t" + c for c in cons)
    return f"""block []:1 (
	in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
	in F[0, 0, 0, 0] {in_dtype}({R}, {S}, {K}, {C}):{sF} #untiled
	out O[0, 0, 0, 0]:assign {out_dtype}({N}, {P}, {Q}, {K}):{sO}
) {{
	0:
	block [n:{N}, x:{P}, y:{Q}, i:{R}, j:{S}, c:{C}, k:{K}]:{pts} (
{lines}
		in I[n, {_aff((stride, 'x'), (1, 'i'), -pad)}, {_aff((stride, 'y'), (1, 'j'), -pad)}, c] {in_dtype}(1, 1, 1, 1):{sI}
		in F[i, j, k, c] {in_dtype}(1, 1, 1, 1):{sF} #untiled
		out O[n, x, y, k]:add {out_dtype}(1, 1, 1, 1):{sO}
	) {{
		0: $I = load(I)
		1: $F = load(F)
		2: $O = mul($I, $F)
		3: O = store($O)
	}}
}}
""".replace("\n\n", "\n")


def conv_fused(N, H, W, C, K, R=3, S=3, stride=1, pad=1, relu=True, residual=False, out_dtype="i8", lo=0):
    """One conv layer in the fused/localized form (conv_layer): O = wrap(max(conv + Bias (+ Res), 0))."""
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    I = Buf("I", "i8", (N, H, W, C))
    F = Buf("F", "i8", (R, S, K, C), tag="untiled")
    B = Buf("Bias", "i32", (K,))
    O = Buf("O", out_dtype, (N, P, Q, K))
    Rz = Buf("Res", "i8", (N, P, Q, K)) if residual else None
    body, _ = conv_layer(I, O, F, B, N, H, W, C, K, R, S, stride, pad, relu, Rz, ind=1, lo=lo)
    refs = [I.ref("in"), F.ref("in"), B.ref("in")] + ([Rz.ref("in")] if Rz else []) + [O.ref("out", agg="assign")]
    return "\n".join(["block []:1 ("] + [f"\t{r}" for r in refs] + [") {", "\t0:", f"\t{body}", "}", ""])


def maxpool2x2(N, H, W, C, dtype="i32"):
    sI = (H * W * C, W * C, C, 1)
    sO = (H // 2 * W // 2 * C, W // 2 * C, C, 1)
    return f"""block []:1 (
	in I[0, 0, 0, 0] {dtype}({N}, {H}, {W}, {C}):{sI}
	out O[0, 0, 0, 0]:assign {dtype}({N}, {H // 2}, {W // 2}, {C}):{sO}
) {{
	0:
	block [n:{N}, x:{H // 2}, y:{W // 2}, c:{C}, i:2, j:2]:{N * H * W * C} (
		in I[n, 2*x + i, 2*y + j, c] {dtype}(1, 1, 1, 1):{sI}
		out O[n, x, y, c]:max {dtype}(1, 1, 1, 1):{sO}
	) {{
		0: $v = load(I)
		1: O = store($v)
	}}
}}
"""


def global_sum(N, H, W, C, in_dtype="i32", out_dtype="i32"):
    sI = (H * W * C, W * C, C, 1)
    return f"""block []:1 (
	in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
	out O[0, 0]:assign {out_dtype}({N}, {C}):({C}, 1)
) {{
	0:
	block [n:{N}, x:{H}, y:{W}, c:{C}]:{N * H * W * C} (
		in I[n, x, y, c] {in_dtype}(1, 1, 1, 1):{sI}
		out O[n, c]:add {out_dtype}(1, 1):({C}, 1)
	) {{
		0: $v = load(I)
		1: O = store($v)
	}}
}}
"""


def conv_useful_macs(N, H, W, C, K, R=3, S=3, pad=1):
    """Constraint-satisfying leaf points (count_valid_points, tile.cpp:338-370), closed form."""
    def axis(L, T):
        return sum(1 for x in range(L) for t in range(T) if 0 <= x + t - pad < L)
    return N * axis(H, R) * axis(W, S) * C * K


def shard_range(total, world, rank):
    """Contiguous split of a partitioned (batch) index across ranks: [lo, hi)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def matmul(M, N, K, in_dtype="i32", out_dtype="i32"):
    """gen_matmul (support.cpp:50-77): C[m,n] += A[m,k] * B[k,n], root C:assign."""
    return f"""block []:1 (
	in A[0, 0] {in_dtype}({M}, {K}):({K}, 1)
	in B[0, 0] {in_dtype}({K}, {N}):({N}, 1)
	out C[0, 0]:assign {out_dtype}({M}, {N}):({N}, 1)
) {{
	0:
	block [m:{M}, n:{N}, k:{K}]:{M * N * K} (
		in A[m, k] {in_dtype}(1, 1):({K}, 1)
		in B[k, n] {in_dtype}(1, 1):({N}, 1)
		out C[m, n]:add {out_dtype}(1, 1):({N}, 1)
	) {{
		0: $a = load(A)
		1: $b = load(B)
		2: $p = mul($a, $b)
		3: C = store($p)
	}}
}}
"""


def conv_bias_relu(N, H, W, C, K, tx=2, in_dtype="i8", acc_dtype="i32", out_dtype="i32"):
    """BASELINE config 3: the conv_relu.stripe structure after tile -> fuse -> localize
    (test_passes.cpp:357-379), with a batch index and a bias add in the ReLU block:
    an outer block over (n, row tiles) owns the per-iteration local accumulator T;
    statement 0 is the 3x3 conv into T, statement 1 is O = max(T + Bias, 0)."""
    assert H % tx == 0
    sI = (H * W * C, W * C, C, 1)
    sF = (3 * K * C, K * C, C, 1)
    sO = (H * W * K, W * K, K, 1)
    sT = (W * K, K, 1)
    xt = H // tx
    return f"""block []:1 (
	in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
	in F[0, 0, 0, 0] {in_dtype}(3, 3, {K}, {C}):{sF} #untiled
	in Bias[0] {acc_dtype}({K}):(1)
	out O[0, 0, 0, 0]:assign {out_dtype}({N}, {H}, {W}, {K}):{sO}
) {{
	0:
	block [n:{N}, x:{xt}]:{N * xt} (
		in I[n, {tx}*x - 1, -1, 0] {in_dtype}(1, {tx + 2}, {W + 2}, {C}):{sI}
		in F[0, 0, 0, 0] {in_dtype}(3, 3, {K}, {C}):{sF} #untiled
		in Bias[0] {acc_dtype}({K}):(1)
		inout T[0, 0, 0]:add {acc_dtype}({tx}, {W}, {K}):{sT}
		out O[n, {tx}*x, 0, 0]:assign {out_dtype}(1, {tx}, {W}, {K}):{sO}
	) {{
		0:
		block [x:{tx}, y:{W}, i:3, j:3, c:{C}, k:{K}, xo={tx}*x]:{tx * W * 9 * C * K} (
			i + x + xo - 1 >= 0
			-i - x - xo + {H} >= 0
			j + y - 1 >= 0
			-j - y + {W} >= 0
			in I[0, x + i, y + j, c] {in_dtype}(1, 1, 1, 1):{sI}
			in F[i, j, k, c] {in_dtype}(1, 1, 1, 1):{sF} #untiled
			out T[x, y, k]:add {acc_dtype}(1, 1, 1):{sT}
		) {{
			0: $I = load(I)
			1: $F = load(F)
			2: $O = mul($I, $F)
			3: T = store($O)
		}}
		1:
		block [x:{tx}, y:{W}, k:{K}]:{tx * W * K} (
			in T[x, y, k] {acc_dtype}(1, 1, 1):{sT}
			in Bias[k] {acc_dtype}(1):(1)
			out O[0, x, y, k]:assign {out_dtype}(1, 1, 1, 1):{sO}
		) {{
			0: $t = load(T)
			1: $b = load(Bias)
			2: $s = add($t, $b)
			3: $z = constant(0)
			4: $r = max($s, $z)
			5: O = store($r)
		}}
	}}
}}
"""


def conv_relu_prefuse(N, H, W, C, K, in_dtype="i8", acc_dtype="i32", out_dtype="i32"):
    """testdata/conv_relu.stripe's structure at config-3 scale, BEFORE the pass pipeline: a
    wrapper block owning T, statement 0 the 3x3 conv leaf [n, x, y, i, j, c, k] into T (add),
    statement 1 the ReLU leaf [n, x, y, k] with a bias, O = max(T + Bias[k], 0).  Config 3 is
    this program after the reference's own autotile -> fuse -> localize -> scalarize
    (test_passes.cpp:357-379), see C3_PIPELINE."""
    sI = (H * W * C, W * C, C, 1)
    sF = (3 * K * C, K * C, C, 1)
    sO = (H * W * K, W * K, K, 1)
    pts = N * H * W * 9 * C * K
    return f"""block []:1 (
	in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
	in F[0, 0, 0, 0] {in_dtype}(3, 3, {K}, {C}):{sF} #untiled
	in Bias[0] {acc_dtype}({K}):(1)
	out O[0, 0, 0, 0]:assign {out_dtype}({N}, {H}, {W}, {K}):{sO}
) {{
	0:
	block []:1 (
		in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
		in F[0, 0, 0, 0] {in_dtype}(3, 3, {K}, {C}):{sF} #untiled
		in Bias[0] {acc_dtype}({K}):(1)
		inout T[0, 0, 0, 0]:assign {acc_dtype}({N}, {H}, {W}, {K}):{sO}
		out O[0, 0, 0, 0]:assign {out_dtype}({N}, {H}, {W}, {K}):{sO}
	) {{
		0:
		block [n:{N}, x:{H}, y:{W}, i:3, j:3, c:{C}, k:{K}]:{pts} (
			i + x - 1 >= 0
			-i - x + {H} >= 0
			j + y - 1 >= 0
			-j - y + {W} >= 0
			in I[n, x + i - 1, y + j - 1, c] {in_dtype}(1, 1, 1, 1):{sI}
			in F[i, j, k, c] {in_dtype}(1, 1, 1, 1):{sF} #untiled
			out T[n, x, y, k]:add {acc_dtype}(1, 1, 1, 1):{sO}
		) {{
			0: $I = load(I)
			1: $F = load(F)
			2: $O = mul($I, $F)
			3: T = store($O)
		}}
		1:
		block [n:{N}, x:{H}, y:{W}, k:{K}]:{N * H * W * K} (
			in T[n, x, y, k] {acc_dtype}(1, 1, 1, 1):{sO}
			in Bias[k] {acc_dtype}(1):(1)
			out O[n, x, y, k]:assign {out_dtype}(1, 1, 1, 1):{sO}
		) {{
			0: $t = load(T)
			1: $b = load(Bias)
			2: $s = add($t, $b)
			3: $z = constant(0)
			4: $r = max($s, $z)
			5: O = store($r)
		}}
	}}
}}
"""


# The pass pipeline of test_passes.cpp:357-379 at config-3 scale (the reference's hwconfig
# syntax, hwconfig.cpp:81-194): tile both kernels per (image, 2-row band), fuse them, localize
# T into the fused block, scalarize.  SRAM sized for one band's working set.
C3_PIPELINE = """mem SRAM cap=1048576 line=64 banks=1
pass autotile unit=SRAM tiles=n:1,x:2 block=0.0
pass autotile unit=SRAM tiles=n:1,x:2 block=0.1
pass fuse block=0 i=0 j=1
pass localize
pass scalarize
pass schedule unit=SRAM
"""


def matmul_bt(M, N, K, in_dtype="i8", out_dtype="i32"):
    """C[m,n] += A[m,k] * B[n,k] (B stored k-contiguous, i.e. transposed)."""
    return matmul(M, N, K, in_dtype, out_dtype).replace(
        f"in B[0, 0] {in_dtype}({K}, {N}):({N}, 1)", f"in B[0, 0] {in_dtype}({N}, {K}):({K}, 1)").replace(
        f"in B[k, n] {in_dtype}(1, 1):({N}, 1)", f"in B[n, k] {in_dtype}(1, 1):({K}, 1)")


# ---- composable program builder (config 5: ResNet-50 and single conv layers) -------------

def _tup(xs):
    return "(" + ", ".join(str(x) for x in xs) + ")"


def _dense(shape):
    st, acc = [], 1
    for d in reversed(shape):
        st.append(acc)
        acc *= d
    return tuple(reversed(st))


def _aff(*terms):
    """Affine text from (coef, name) / int terms, e.g. _aff((2, 'x'), (1, 'i'), -3) -> '2*x + i - 3'."""
    out = []
    const = 0
    for t in terms:
        if isinstance(t, int):
            const += t
            continue
        k, n = t
        if k == 0:
            continue
        s = n if abs(k) == 1 else f"{abs(k)}*{n}"
        out.append(("- " if k < 0 else "+ ") + s)
    if const:
        out.append(("- " if const < 0 else "+ ") + str(abs(const)))
    if not out:
        return "0"
    txt = " ".join(out)
    return txt[2:] if txt.startswith("+ ") else "-" + txt[2:]


class Buf:
    def __init__(self, name, dtype, shape, tag=""):
        self.name, self.dtype, self.shape, self.tag = name, dtype, tuple(shape), tag
        self.strides = _dense(shape)

    @property
    def elements(self):
        n = 1
        for s in self.shape:
            n *= s
        return n

    def ref(self, direction, offsets=None, agg=None, sizes=None):
        offs = offsets if offsets is not None else ["0"] * len(self.shape)
        a = f":{agg}" if agg else ""
        sz = sizes if sizes is not None else self.shape
        tag = f" #{self.tag}" if self.tag else ""
        return f"{direction} {self.name}[{', '.join(offs)}]{a} {self.dtype}{_tup(sz)}:{_tup(self.strides)}{tag}"

    def point(self, direction, offsets, agg=None):
        return self.ref(direction, offsets, agg, sizes=[1] * len(self.shape))


def _block(idx, cons, refs, body, ind):
    """idx: list of (name, range) or alias strings."""
    pts = 1
    names = []
    for i in idx:
        if isinstance(i, tuple):
            names.append(f"{i[0]}:{i[1]}")
            pts *= i[1]
        else:
            names.append(i)
    t = "\t" * ind
    lines = [f"block [{', '.join(names)}]:{pts} ("]
    lines += [f"{t}\t{c}" for c in cons]
    lines += [f"{t}\t{r}" for r in refs]
    lines.append(f"{t}) {{")
    for k, s in enumerate(body):
        if s.startswith("block"):
            lines.append(f"{t}\t{k}:")
            lines.append(f"{t}\t{s}")
        else:
            lines.append(f"{t}\t{k}: {s}")
    lines.append(f"{t}}}")
    return "\n".join(lines)


def conv_layer(src, dst, w, b, N, H, W, C, K, R, S, stride, pad, relu=True, residual=None, ind=1,
               acc_dtype="i32", tname="T", lo=0):
    """One conv + bias (+ residual) (+ ReLU) as the fuse/localize passes leave it
    (test_passes.cpp:357-379): a wrapper block owning the local accumulator T,
    statement 0 the conv leaf into T (add), statement 1 the element-wise epilogue
    writing dst (assign)."""
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    T = Buf(tname, acc_dtype, (N, P, Q, K))
    cons = []
    if pad:
        # padding halo: the input row/col of every counted tap lies inside the image
        cons.append(f"{_aff((stride, 'x'), (1, 'i'), -pad)} >= 0")
        cons.append(f"{_aff((-stride, 'x'), (-1, 'i'), H - 1 + pad)} >= 0")
        cons.append(f"{_aff((stride, 'y'), (1, 'j'), -pad)} >= 0")
        cons.append(f"{_aff((-stride, 'y'), (-1, 'j'), W - 1 + pad)} >= 0")
    conv_refs = [src.point("in", ["n", _aff((stride, "x"), (1, "i"), -pad), _aff((stride, "y"), (1, "j"), -pad), "c"]),
                 w.point("in", ["i", "j", "k", "c"]),
                 T.point("out", ["n", "x", "y", "k"], "add")]
    conv = _block([("n", N), ("x", P), ("y", Q), ("i", R), ("j", S), ("c", C), ("k", K)], cons, conv_refs,
                  [f"$I = load({src.name})", f"$F = load({w.name})", "$O = mul($I, $F)", f"{T.name} = store($O)"],
                  ind + 1)
    epi_refs = [T.point("in", ["n", "x", "y", "k"]), b.point("in", ["k"])]
    body = [f"$t = load({T.name})", f"$b = load({b.name})", "$s = add($t, $b)"]
    v = "$s"
    if residual is not None:
        epi_refs.append(residual.point("in", ["n", "x", "y", "k"]))
        body += [f"$r = load({residual.name})", "$u = add($s, $r)"]
        v = "$u"
    if relu:
        body += [f"$z = constant({lo})", f"$o = max({v}, $z)"]
        v = "$o"
    epi_refs.append(dst.point("out", ["n", "x", "y", "k"], "assign"))
    body.append(f"{dst.name} = store({v})")
    epi = _block([("n", N), ("x", P), ("y", Q), ("k", K)], [], epi_refs, body, ind + 1)
    outer_refs = [src.ref("in"), w.ref("in"), b.ref("in")]
    if residual is not None:
        outer_refs.append(residual.ref("in"))
    outer_refs += [T.ref("inout", agg="add"), dst.ref("out", agg="assign")]
    return _block([], [], outer_refs, [conv, epi], ind), (P, Q)


def resnet50(N, image=224, width=64, stages=(3, 4, 6, 3), classes=1000, in_ch=3):
    """BASELINE config 5: a ResNet-50 v1.5-shaped Stripe program.

    Integer semantics throughout (the reference has no float): i8 activations and
    weights, i32 accumulators and biases, ReLU outputs stored to i8 (wrapping, ir.cpp:39-48).
    Layers: 7x7/2 stem conv + bias + ReLU, 3x3/2 max-pool (padding constraints),
    bottleneck stages (1x1 -> 3x3 (stride on the 3x3, v1.5) -> 1x1, projection 1x1 on the
    first block of each stage, residual add + ReLU), global 7x7 sum (no divide intrinsic;
    the 1/49 folds into fc), fc matmul + bias.  Activations are locals of one top-level
    network block (device-resident scratch); the program's buffers are the image, the
    weights and the logits.  Returns (text, info) with per-conv shapes and useful MACs.
    """
    bufs_in, locals_, body, convs = [], [], [], []
    X = Buf("X", "i8", (N, image, image, in_ch))
    bufs_in.append(X)
    lid = [0]

    def new_conv(src, H, W, C, K, R, S, stride, pad, relu=True, residual=None):
        l = lid[0]
        lid[0] += 1
        w = Buf(f"W{l}", "i8", (R, S, K, C), tag="untiled")
        b = Buf(f"B{l}", "i32", (K,))
        bufs_in.extend([w, b])
        P = (H + 2 * pad - R) // stride + 1
        Q = (W + 2 * pad - S) // stride + 1
        dst = Buf(f"A{l}", "i8", (N, P, Q, K))
        locals_.append(dst)
        txt, _ = conv_layer(src, dst, w, b, N, H, W, C, K, R, S, stride, pad, relu, residual, ind=2,
                            tname=f"T{l}")
        body.append(txt)
        macs = N * K * C * sum(1 for x in range(P) for i in range(R) if 0 <= stride * x + i - pad < H) * \
            sum(1 for y in range(Q) for j in range(S) if 0 <= stride * y + j - pad < W)
        convs.append(dict(layer=l, H=H, W=W, C=C, K=K, R=R, S=S, stride=stride, pad=pad, P=P, Q=Q, macs=macs,
                          residual=residual is not None))
        return dst, P, Q

    a, H, W = new_conv(X, image, image, in_ch, width, 7, 7, 2, 3)
    # 3x3/2 max-pool with padding constraints into a zero-initialised local
    P = (H + 2 - 3) // 2 + 1
    pool = Buf("Pool", "i8", (N, P, P, width))
    locals_.append(pool)
    cons = [f"{_aff((2, 'x'), (1, 'i'), -1)} >= 0", f"{_aff((-2, 'x'), (-1, 'i'), H)} >= 0",
            f"{_aff((2, 'y'), (1, 'j'), -1)} >= 0", f"{_aff((-2, 'y'), (-1, 'j'), W)} >= 0"]
    body.append(_block([("n", N), ("x", P), ("y", P), ("c", width), ("i", 3), ("j", 3)], cons,
                       [a.point("in", ["n", _aff((2, "x"), (1, "i"), -1), _aff((2, "y"), (1, "j"), -1), "c"]),
                        pool.point("out", ["n", "x", "y", "c"], "max")],
                       [f"$v = load({a.name})", f"{pool.name} = store($v)"], 2))
    a, H, W, C = pool, P, P, width
    for si, nblocks in enumerate(stages):
        mid = width * (2 ** si)
        out = mid * 4
        for bi in range(nblocks):
            stride = 2 if (bi == 0 and si > 0) else 1
            if bi == 0:
                sc, _, _ = new_conv(a, H, W, C, out, 1, 1, stride, 0, relu=False)
            else:
                sc = a
            t1, H1, W1 = new_conv(a, H, W, C, mid, 1, 1, 1, 0)
            t2, H2, W2 = new_conv(t1, H1, W1, mid, mid, 3, 3, stride, 1)
            a, H, W = new_conv(t2, H2, W2, mid, out, 1, 1, 1, 0, relu=True, residual=sc)
            C = out
    # global sum over the final H x W (wraps into i8 like every activation store)
    G = Buf("G", "i8", (N, C))
    locals_.append(G)
    body.append(_block([("n", N), ("x", H), ("y", W), ("c", C)], [],
                       [a.point("in", ["n", "x", "y", "c"]), G.point("out", ["n", "c"], "add")],
                       [f"$v = load({a.name})", f"{G.name} = store($v)"], 2))
    Wfc = Buf("Wfc", "i8", (classes, C), tag="untiled")
    Bfc = Buf("Bfc", "i32", (classes,))
    bufs_in.extend([Wfc, Bfc])
    logits = Buf("Logits", "i32", (N, classes))
    Tfc = Buf("Tfc", "i32", (N, classes))
    fc = _block([("n", N), ("o", classes), ("c", C)], [],
                [G.point("in", ["n", "c"]), Wfc.point("in", ["o", "c"]), Tfc.point("out", ["n", "o"], "add")],
                [f"$g = load({G.name})", f"$w = load({Wfc.name})", "$p = mul($g, $w)", f"{Tfc.name} = store($p)"], 3)
    fce = _block([("n", N), ("o", classes)], [],
                 [Tfc.point("in", ["n", "o"]), Bfc.point("in", ["o"]), logits.point("out", ["n", "o"], "assign")],
                 [f"$t = load({Tfc.name})", f"$b = load({Bfc.name})", "$s = add($t, $b)",
                  f"{logits.name} = store($s)"], 3)
    body.append(_block([], [], [G.ref("in"), Wfc.ref("in"), Bfc.ref("in"), Tfc.ref("inout", agg="add"),
                                logits.ref("out", agg="assign")], [fc, fce], 2))
    net_refs = [x.ref("in") for x in bufs_in] + [logits.ref("out", agg="assign")]
    net_refs += [l.ref("inout", agg="assign") for l in locals_]
    net = _block([], [], net_refs, body, 1)
    root_refs = [x.ref("in") for x in bufs_in] + [logits.ref("out", agg="assign")]
    text = "\n".join([f"block []:1 ("] + [f"\t{r}" for r in root_refs] + [") {", "\t0:", f"\t{net}", "}", ""])
    macs = sum(c["macs"] for c in convs) + N * classes * C
    info = dict(convs=convs, macs=macs, flops=2 * macs, inputs=[x.name for x in bufs_in], output="Logits")
    return text, info


def pool2d(N, H, W, C, R=3, S=3, stride=2, pad=1, agg="max", dtype="i8"):
    """Windowed max/min with padding constraints (the ResNet stem pool shape)."""
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    I = Buf("I", dtype, (N, H, W, C))
    O = Buf("O", dtype, (N, P, Q, C))
    cons = []
    if pad:
        cons = [f"{_aff((stride, 'x'), (1, 'i'), -pad)} >= 0", f"{_aff((-stride, 'x'), (-1, 'i'), H - 1 + pad)} >= 0",
                f"{_aff((stride, 'y'), (1, 'j'), -pad)} >= 0", f"{_aff((-stride, 'y'), (-1, 'j'), W - 1 + pad)} >= 0"]
    blk = _block([("n", N), ("x", P), ("y", Q), ("c", C), ("i", R), ("j", S)], cons,
                 [I.point("in", ["n", _aff((stride, "x"), (1, "i"), -pad), _aff((stride, "y"), (1, "j"), -pad), "c"]),
                  O.point("out", ["n", "x", "y", "c"], agg)],
                 ["$v = load(I)", "O = store($v)"], 1)
    return "\n".join(["block []:1 (", f"\t{I.ref('in')}", f"\t{O.ref('out', agg='assign')}", ") {", "\t0:",
                      f"\t{blk}", "}", ""])
