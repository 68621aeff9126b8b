"""The tcgen05 decode GEMM (decode_gemm.cu) against a
plain PyTorch reference of the same op (y = x W^T in float64 on the same bf16
values): ragged N, K and batch, forced and planned K splits, every batch width
the kernel instantiates (N side 32 / 64 / 128 / 256). The split slices must sum
to the product and each slice must be the product over its own K range. GPU only."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def ref(w, x):
    return x.double() @ w.double().T


@pytest.mark.parametrize("N,K,B,splits", [
    (256, 256, 4, 1), (128, 64, 1, 1), (1000, 776, 37, 0), (1000, 776, 37, 3), (5120, 5120, 64, 0),
    (15360, 5120, 29, 0), (4096, 14336, 64, 0), (8192, 1024, 64, 0), (512, 1024, 256, 2), (700, 2048, 200, 0),
    (384, 4096, 16, 16), (130, 520, 130, 0)])
def test_decode_gemm_matches_reference(N, K, B, splits):
    from paper_2507_11507_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K * 3 + B)
    w = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    y, ns = _lib.decode_gemm(w, x, splits)
    torch.cuda.synchronize()
    assert ns >= 1 and (splits == 0 or ns == splits)
    r = ref(w, x)
    got = y.double().sum(0)
    scale = r.abs().max().item()
    assert (got - r).abs().max().item() <= 2e-5 * scale + 1e-6 * K ** 0.5
    # each slice is the product over its own K range (64-wide blocks, split in order)
    n_kb = (K + 63) // 64
    per = (n_kb + ns - 1) // ns
    for s in range(ns):
        k0, k1 = min(K, s * per * 64), min(K, (s + 1) * per * 64)
        rs = ref(w[:, k0:k1], x[:, k0:k1]) if k1 > k0 else torch.zeros_like(r)
        assert (y[s].double() - rs).abs().max().item() <= 2e-5 * scale + 1e-6 * K ** 0.5


@pytest.mark.parametrize("N,K,B,splits", [(5120, 5120, 64, 0), (1000, 776, 37, 3), (8192, 1024, 128, 4),
                                          (384, 4096, 16, 8), (700, 2048, 100, 0), (4096, 14336, 64, 2)])
def test_decode_gemm_cluster_reduce_equals_the_slice_sum(N, K, B, splits):
    """reduce: the K splits of a tile are summed inside the kernel through the
    cluster's distributed shared memory, in split order -- bit-identical to
    summing the unreduced slices in slice order, as the residual kernel does."""
    from paper_2507_11507_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(N + K + B)
    w = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    s_plain, ns = _lib.decode_gemm(w, x, splits)
    s_red, one = _lib.decode_gemm(w, x, min(ns, 8) if splits == 0 else splits, reduce=True)
    torch.cuda.synchronize()
    assert one == 1
    if splits == 0:
        s_plain, ns = _lib.decode_gemm(w, x, min(ns, 8))
    acc = s_plain[0].clone()
    for i in range(1, ns):
        acc += s_plain[i]
    assert torch.equal(s_red[0], acc)
    r = ref(w, x)
    assert (s_red[0].double() - r).abs().max().item() <= 2e-5 * r.abs().max().item() + 1e-6 * K ** 0.5


def test_decode_gemm_is_deterministic():
    from paper_2507_11507_b200 import _lib
    w = torch.randn((4096, 4096), device="cuda").to(torch.bfloat16)
    x = torch.randn((64, 4096), device="cuda").to(torch.bfloat16)
    a, _ = _lib.decode_gemm(w, x)
    b, _ = _lib.decode_gemm(w, x)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


SK_SHAPES = [(5120, 5120, 64), (8192, 1024, 64), (15360, 5120, 29), (1000, 776, 37), (130, 520, 130),
             (20480, 5120, 16), (512, 1024, 256), (128, 64, 1), (700, 2048, 200), (1280, 8192, 64),
             (8192, 3584, 33), (256, 64, 8)]


@pytest.mark.parametrize("N,K,B", SK_SHAPES)
def test_sk_gemm_matches_reference(N, K, B):
    """Persistent stream-K form: tiles cut between CTAs are finished in the GEMM
    (owner adds the parked partials in K order). One fp32 output vs fp64 torch,
    and bit-identical across runs (deterministic fixup)."""
    from paper_2507_11507_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(N * 5 + K * 11 + B)
    w = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    y = _lib.sk_gemm(w, x)
    y2 = _lib.sk_gemm(w, x)
    torch.cuda.synchronize()
    r = ref(w, x)
    scale = r.abs().max().item()
    assert (y.double() - r).abs().max().item() <= 2e-5 * scale + 1e-6 * K ** 0.5
    assert torch.equal(y, y2)


@pytest.mark.parametrize("N,K,B,relu", [(20480, 5120, 64, True), (1000, 776, 37, True), (4096, 4096, 200, False)])
def test_sk_gemm_bias_relu_bf16_epilogue(N, K, B, relu):
    """The column-parallel epilogue (FC1: + bias, ReLU, bf16 store) inside the GEMM."""
    from paper_2507_11507_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K + 7 * B)
    w = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    bias = (torch.randn((N,), generator=g, device="cuda") * 0.1).to(torch.bfloat16)
    y32 = _lib.sk_gemm(w, x, bias=bias, relu=relu)
    y16 = _lib.sk_gemm(w, x, bias=bias, relu=relu, out_bf16=True)
    torch.cuda.synchronize()
    r = ref(w, x) + bias.double()
    if relu:
        r = r.clamp_min(0)
    scale = r.abs().max().item()
    assert (y32.double() - r).abs().max().item() <= 2e-5 * scale + 1e-6 * K ** 0.5
    assert torch.equal(y16, y32.to(torch.bfloat16))          # the same value, rounded once


@pytest.mark.parametrize("N,K,B,splits,cg", [(8192, 1024, 64, 1, 2), (8192, 3584, 64, 1, 2), (1000, 776, 37, 1, 2),
                                             (700, 2048, 200, 1, 4), (8192, 1024, 128, 1, 4), (384, 4096, 16, 1, 2),
                                             (5120, 5120, 100, 3, 3), (130, 520, 250, 2, 8),
                                             (5120, 1024, 400, 1, 2), (1000, 776, 300, 2, 4)])
def test_decode_gemm_column_groups_bit_identical(N, K, B, splits, cg):
    """col_groups: the batch rows are cut into groups, one CTA per (tile, split,
    group), each re-reading its tile's weights. Every output element still sums the
    same K blocks in the same MMA order, so the slices are bit-identical to the
    ungrouped launch, and within the fp64 reference's bound. Ragged groups (B not a
    multiple of the group width) and groups that round to an empty tail included;
    with groups the batch may exceed one MMA's 256 columns (B = 300, 400)."""
    from paper_2507_11507_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(N * 5 + K + B * 11 + cg)
    w = (torch.randn((N, K), generator=g, device="cuda") / K ** 0.5).to(torch.bfloat16)
    x = torch.randn((B, K), generator=g, device="cuda").to(torch.bfloat16)
    yg, ng = _lib.decode_gemm(w, x, splits, col_groups=cg)
    torch.cuda.synchronize()
    assert ng == splits
    r = ref(w, x)
    got = yg.double().sum(0)
    assert (got - r).abs().max().item() <= 2e-5 * r.abs().max().item() + 1e-6 * K ** 0.5
    if B > 256:  # more rows than one MMA's N: only a grouped launch exists
        with pytest.raises(_lib.MirageError):
            _lib.decode_gemm(w, x, splits)
        return
    y1, n1 = _lib.decode_gemm(w, x, splits)
    torch.cuda.synchronize()
    assert n1 == splits
    # the group width is rounded to 32/64/128/256 rows, so the MMA N differs between
    # the two launches: compare element values, which tcgen05 accumulates per column
    assert torch.equal(yg, y1)
