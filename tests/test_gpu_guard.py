"""Out-of-bounds writes, checked without compute-sanitizer (closed on this pool): every output
buffer sits inside a larger allocation whose guard bands before and after are filled with a sentinel; after the
kernel the bands must be untouched.  Ragged shapes (M, N, K not multiples of the tiles, M not a multiple of 4,
odd element counts) so every kernel's tail path writes at the edge of its buffer."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SENT = -12345.0
PAD = 4096   # floats on each side (16 KB), a multiple of 4 so the buffer stays 16-B aligned


@pytest.fixture(scope="module")
def pz():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1512_06216_b200 as pz
    return pz


def guarded(n, fill=None):
    big = torch.full((n + 2 * PAD,), SENT, device="cuda")
    view = big[PAD:PAD + n]
    if fill is not None:
        view.copy_(fill.reshape(-1))
    return big, view


def bands_intact(big, n):
    torch.cuda.synchronize()
    return bool((big[:PAD] == SENT).all()) and bool((big[PAD + n:] == SENT).all())


@pytest.mark.parametrize("M,N,K,P", [(300, 520, 40, 2), (1000, 4100, 37, 3), (4, 4, 1, 1), (257, 260, 33, 1)])
@pytest.mark.parametrize("recon", ["tf32", "fp32"])
def test_k1_writes_stay_inside_w(pz, M, N, K, P, recon):
    ldk = (K + 3) // 4 * 4
    Ug = torch.zeros(P, M, ldk, device="cuda")
    Vg = torch.zeros(P, N, ldk, device="cuda")
    Ug[:, :, :K] = torch.randn(P, M, K, device="cuda")
    Vg[:, :, :K] = torch.randn(P, N, K, device="cuda")
    big, w = guarded(M * N, torch.randn(M, N, device="cuda"))
    pz.reconstruct_sgd(Ug, Vg, P, K, ldk, M, N, w.view(M, N), -1e-3,
                       recon=pz.RECON_TF32 if recon == "tf32" else pz.RECON_FP32)
    assert bands_intact(big, M * N)


@pytest.mark.parametrize("M,N,K,P", [(300, 520, 40, 2), (1000, 4096, 37, 1), (4, 4, 1, 1)])
def test_k1_mn_writes_stay_inside_w(pz, M, N, K, P):
    Mp = (M + 3) // 4 * 4
    U = torch.randn(P, K, Mp, device="cuda")
    V = torch.randn(P, K, N, device="cuda")
    big, w = guarded(M * N, torch.randn(M, N, device="cuda"))
    pz.reconstruct_sgd_mn(U, V, P, K, M, N, w.view(M, N), -1e-3)
    assert bands_intact(big, M * N)


@pytest.mark.parametrize("n", [1, 3, 4097, 10_007, 1_000_003])
def test_k2_writes_stay_inside_w(pz, n):
    g = torch.randn(n, device="cuda")
    big, w = guarded(n, torch.randn(n, device="cuda"))
    pz.ps_shard_update(g, w, n, -1e-3)
    assert bands_intact(big, n)


@pytest.mark.parametrize("M,N,K", [(300, 520, 40), (1000, 4100, 300), (5, 7, 3)])
def test_k3_pack_writes_stay_inside_slots(pz, M, N, K):
    ldk = (K + 3) // 4 * 4
    U = torch.randn(K, M, device="cuda")
    V = torch.randn(K, N, device="cuda")
    bu, u = guarded(M * ldk)
    bv, v = guarded(N * ldk)
    bs, cs = guarded(M)
    pz.pack_factors(U, V, K, ldk, u, v, cs)
    assert bands_intact(bu, M * ldk) and bands_intact(bv, N * ldk) and bands_intact(bs, M)
