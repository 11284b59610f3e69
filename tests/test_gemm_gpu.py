"""GPU: tcgen05 GEMM (csrc/gemm.cu) vs a plain PyTorch fp32 reference."""
import pytest
import torch

from paper_2507_07966_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["1", "2", "3"], autouse=True)
def gemm_impl(request, monkeypatch):
    """Every kernel variant (MRSP_GEMM_IMPL): single CTA, CTA pair with the
    2-SM TMA form, CTA pair with relayed stage completion."""
    monkeypatch.setenv("MRSP_GEMM_IMPL", request.param)
    return request.param


def ref(A, B):
    return A.float() @ B.float().T


def rel_err(x, y):
    return ((x.float() - y.float()).norm() / (y.float().norm() + 1e-12)).item()


SHAPES = [(128, 256, 64), (256, 512, 128), (300, 700, 200), (1000, 1152, 1152), (77, 4608, 3584),
          (4096, 4096, 4096), (515, 32, 256), (16384, 1152, 592)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_store(gpu, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    C = ops.gemm(A, B, ops.EPI_STORE_F32)
    torch.cuda.synchronize()
    assert rel_err(C, ref(A, B)) < 1e-5
    Cb = ops.gemm(A, B)
    assert rel_err(Cb, ref(A, B)) < 5e-3


def test_gemm_epilogues(gpu):
    M, N, K = 300, 512, 320
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda")
    r = ref(A, B)
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_BF16, bias=bias), r + bias) < 5e-3
    gelu = torch.nn.functional.gelu(r + bias, approximate="tanh")
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_GELU_BF16, bias=bias), gelu) < 5e-3
    resid = torch.randn(M, N, device="cuda")
    want = resid + r
    ops.gemm(A, B, ops.EPI_RESID_F32, resid=resid)
    assert rel_err(resid, want) < 1e-5
    resid2 = torch.randn(M, N, device="cuda")
    want2 = resid2 + r + bias
    ops.gemm(A, B, ops.EPI_RESID_F32, resid=resid2, bias=bias)
    assert rel_err(resid2, want2) < 1e-5
    out = ops.gemm(A, B, ops.EPI_SWIGLU_BF16)
    rr = r.view(M, N // 256, 2, 128)
    sw = (torch.nn.functional.silu(rr[:, :, 0]) * rr[:, :, 1]).reshape(M, N // 2)
    assert rel_err(out, sw) < 5e-3


def test_gemm_strided_operands(gpu):
    # A is a column slice of a wider buffer (e.g. one head of a packed QKV).
    X = torch.randn(512, 1024, device="cuda").bfloat16()
    A = X[:, 256:768]
    B = torch.randn(384, 512, device="cuda").bfloat16()
    assert rel_err(ops.gemm(A, B, ops.EPI_STORE_F32), ref(A, B)) < 1e-5


# Decode-shaped GEMMs (M = G rows): split-K over the SMs with a workspace,
# every plain epilogue, against the fp32 reference and the unsplit kernel.
SPLITK = [(8, 4608, 3584), (8, 3584, 3584), (8, 3584, 18944), (1, 1152, 4304), (77, 640, 2048),
          (128, 512, 8192), (8, 37888, 3584)]


@pytest.mark.parametrize("M,N,K", SPLITK)
def test_gemm_splitk_epilogues(gpu, gemm_impl, M, N, K):
    if gemm_impl != "1":
        pytest.skip("split-K is a mode of the single-CTA kernel")
    g = torch.Generator(device="cuda").manual_seed(N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    ws = torch.empty(ops.splitk_workspace_bytes(M), dtype=torch.uint8, device="cuda")
    r = ref(A, B)
    C = ops.gemm(A, B, ops.EPI_STORE_F32, splitk_ws=ws)
    assert rel_err(C, r) < 5e-5  # fp32 sums over K up to 18944 in another order
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_BF16, bias=bias, splitk_ws=ws), r + bias) < 5e-3
    gelu = torch.nn.functional.gelu(r + bias, approximate="tanh")
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_GELU_BF16, bias=bias, splitk_ws=ws), gelu) < 5e-3
    resid = torch.randn(M, N, device="cuda", generator=g)
    want = resid + r + bias
    ops.gemm(A, B, ops.EPI_RESID_F32, resid=resid, bias=bias, splitk_ws=ws)
    assert rel_err(resid, want) < 5e-5
    if N % 256 == 0:
        out = ops.gemm(A, B, ops.EPI_SWIGLU_BF16, splitk_ws=ws)
        rr = r.view(M, N // 256, 2, 128)
        sw = (torch.nn.functional.silu(rr[:, :, 0]) * rr[:, :, 1]).reshape(M, N // 2)
        assert rel_err(out, sw) < 5e-3
    # deterministic: same bits twice; close to the unsplit kernel
    C2 = ops.gemm(A, B, ops.EPI_STORE_F32, splitk_ws=ws)
    assert torch.equal(C, C2)
    assert rel_err(C, ops.gemm(A, B, ops.EPI_STORE_F32)) < 5e-5


@pytest.mark.parametrize("M,N,K", [(8, 4608, 3584), (16, 37888, 3584), (3, 152064, 256)])
def test_gemm_skinny_matches_default(gpu, gemm_impl, M, N, K, monkeypatch):
    """M <= 16: the skinny ring (16-row A boxes, 6 stages) gives the same bits as
    the default 128-row tile for the rows that exist, split or not."""
    if gemm_impl != "1":
        pytest.skip("the skinny ring is a mode of the single-CTA kernel")
    g = torch.Generator(device="cuda").manual_seed(M * N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    ws = torch.empty(ops.splitk_workspace_bytes(M), dtype=torch.uint8, device="cuda")
    out = {}
    for sk in ("0", "1"):
        monkeypatch.setenv("MRSP_GEMM_SKINNY", sk)
        out[sk] = [ops.gemm(A, B, ops.EPI_STORE_F32), ops.gemm(A, B, ops.EPI_STORE_F32, splitk_ws=ws),
                   ops.gemm(A, B, ops.EPI_BIAS_BF16, bias=bias),
                   ops.gemm(A, B, ops.EPI_SWIGLU_BF16) if N % 256 == 0 else None]
    for x, y in zip(out["0"], out["1"]):
        if x is not None:
            assert torch.equal(x, y)
    assert rel_err(out["1"][0], ref(A, B)) < 1e-5


@pytest.mark.parametrize("N", [1152, 3456])
def test_gemm_bn192_epilogues(gpu, gemm_impl, N):
    """N a multiple of 192 but not of 256 (SigLIP's O / fc2 and QKV widths):
    every plain epilogue, with the default tiles and (a subprocess with
    MRSP_GEMM_BN192=1) the 192-wide-tile kernel."""
    M, K = 1300, 1152
    g = torch.Generator(device="cuda").manual_seed(N)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    r = ref(A, B)
    assert rel_err(ops.gemm(A, B, ops.EPI_STORE_F32), r) < 1e-5
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_BF16, bias=bias), r + bias) < 5e-3
    gelu = torch.nn.functional.gelu(r + bias, approximate="tanh")
    assert rel_err(ops.gemm(A, B, ops.EPI_BIAS_GELU_BF16, bias=bias), gelu) < 5e-3
    resid = torch.randn(M, N, device="cuda", generator=g)
    want = resid + r + bias
    ops.gemm(A, B, ops.EPI_RESID_F32, resid=resid, bias=bias)
    assert rel_err(resid, want) < 1e-5


def test_gemm_bn192_variant(gpu):
    """The 192-wide-tile kernel (read once per process) in a subprocess."""
    import os
    import subprocess
    import sys
    code = ("import torch, sys; sys.path.insert(0, '.');"
            "from paper_2507_07966_b200 import ops;"
            "g = torch.Generator(device='cuda').manual_seed(3);"
            "A = torch.randn(1300, 1152, device='cuda', generator=g).bfloat16();"
            "B = (torch.randn(3456, 1152, device='cuda', generator=g) / 34).bfloat16();"
            "bias = torch.randn(3456, device='cuda', generator=g);"
            "r = A.float() @ B.float().T + bias;"
            "C = ops.gemm(A, B, ops.EPI_BIAS_BF16, bias=bias);"
            "R = torch.randn(1300, 3456, device='cuda', generator=g); W = R + r;"
            "ops.gemm(A, B, ops.EPI_RESID_F32, resid=R, bias=bias);"
            "e1 = ((C.float() - r).norm() / r.norm()).item();"
            "e2 = ((R - W).norm() / W.norm()).item();"
            "assert e1 < 5e-3 and e2 < 1e-5, (e1, e2); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env={**os.environ, "MRSP_GEMM_BN192": "1", "MRSP_GEMM_IMPL": "1"},
                         timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
