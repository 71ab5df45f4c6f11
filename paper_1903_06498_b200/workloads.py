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


def conv2d(N, H, W, C, K, R=3, S=3, in_dtype="i8", out_dtype="i32", pad=1):
    """O[n,x,y,k] += I[n, x+i-pad, y+j-pad, c] * F[i,j,k,c], constraints keep taps in bounds."""
    sI = (H * W * C, W * C, C, 1)
    sF = (S * K * C, K * C, C, 1)
    sO = (H * W * K, W * K, K, 1)
    pts = N * H * W * R * S * C * K

    def aff(idx, off):
        if off == 0:
            return f"{idx[1]} + {idx[0]}"
        return f"{idx[1]} + {idx[0]} - {off}" if off > 0 else f"{idx[1]} + {idx[0]} + {-off}"

    cons = []
    if pad:
        cons = [f"i + x - {pad} >= 0", f"-i - x + {H - 1 + pad} >= 0",
                f"j + y - {pad} >= 0", f"-j - y + {W - 1 + pad} >= 0"]
    lines = "\n".join("\t\t" + c for c in cons)
    return f"""block []:1 (
	in I[0, 0, 0, 0] {in_dtype}({N}, {H}, {W}, {C}):{sI}
	in F[0, 0, 0, 0] {in_dtype}({R}, {S}, {K}, {C}):{sF} #untiled
	out O[0, 0, 0, 0]:assign {out_dtype}({N}, {H}, {W}, {K}):{sO}
) {{
	0:
	block [n:{N}, x:{H}, y:{W}, i:{R}, j:{S}, c:{C}, k:{K}]:{pts} (
{lines}
		in I[n, {aff(('x', 'i'), pad)}, {aff(('y', 'j'), pad)}, c] {in_dtype}(1, 1, 1, 1):{sI}
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


def matmul_bt(M, N, K, in_dtype="i8", out_dtype="i32"):
    """C[m,n] += A[m,k] * B[n,k] (B stored k-contiguous, i.e. transposed)."""
    return matmul(M, N, K, in_dtype, out_dtype).replace(
        f"in B[0, 0] {in_dtype}({K}, {N}):({N}, 1)", f"in B[0, 0] {in_dtype}({N}, {K}):({K}, 1)").replace(
        f"in B[k, n] {in_dtype}(1, 1):({N}, 1)", f"in B[n, k] {in_dtype}(1, 1):({K}, 1)")
