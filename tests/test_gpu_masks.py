"""On-device RM/FM sampling-set generators (ifctn_mask_uniform / ifctn_mask_fibres, SURVEY
§8(f3)) against oracle/masks.py: bit-exact masks (-m gpu)."""
import numpy as np
import pytest

from oracle import masks as MK

from gpu_util import requires_cuda, torch

pytestmark = [pytest.mark.gpu, requires_cuda]


def _uniform(n, k, seed):
    from paper_2511_16358_b200 import mask_uniform
    return mask_uniform(n, k, seed).cpu().numpy()


@pytest.mark.parametrize("n", [1, 15, 16, 17, 1000, 100003, 2**20 + 5])
def test_uniform_bit_exact(n):
    for k in sorted({0, 1, n // 20, n // 2, max(n - 1, 0), n}):
        for seed in (0, 1, 2**63 + 11):
            g = _uniform(n, k, seed)
            assert np.array_equal(g, MK.mask_uniform(n, k, seed)), (n, k, seed)


def test_uniform_unaligned_and_stream_ordered():
    from paper_2511_16358_b200 import _abi
    n, k, seed = 4099, 777, 5
    buf = torch.full((n + 3,), 7, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        _abi.ifctn_mask_uniform(buf.data_ptr() + 1, n, k, seed, s.cuda_stream)
    s.synchronize()
    h = buf.cpu().numpy()
    assert h[0] == 7 and h[-2] == 7 and h[-1] == 7     # nothing written outside [1, n+1)
    assert np.array_equal(h[1:n + 1], MK.mask_uniform(n, k, seed))


@pytest.mark.parametrize("dims,mode,missing", [((4, 3, 5), 0, 6), ((4, 3, 5), 1, 11), ((4, 3, 5), 2, 0),
                                               ((4, 3, 5), 2, 12), ((2, 3, 4, 5), 2, 29),
                                               ((7, 9, 11, 13), 3, 300), ((33,), 0, 1),
                                               ((214, 61, 144, 4), 2, 36551)])
def test_fibres_bit_exact(dims, mode, missing):
    from paper_2511_16358_b200 import mask_fibres
    for seed in (0, 3):
        g = mask_fibres(dims, mode, missing, seed).cpu().numpy()
        assert np.array_equal(g, MK.mask_fibres(dims, mode, missing, seed)), (dims, mode, missing, seed)


def test_uniform_full_c5_size():
    """C5's RM draw (64⁴×32, 5%): exact count, and every selected key below every unselected
    key (the defining property of the k smallest), keys from the oracle's stream in chunks."""
    n, k, seed = 64 ** 4 * 32, 26843546, 0
    m = _uniform(n, k, seed)
    assert int(m.sum(dtype=np.int64)) == k
    hi_sel, lo_un = 0, 2 ** 64 - 1
    chunk = 1 << 26
    for c0 in range(0, n, chunk):
        z = MK.splitmix64_keys(seed, min(chunk, n - c0), start=c0)
        sel = m[c0:c0 + z.size].astype(bool)
        if sel.any():
            hi_sel = max(hi_sel, int(z[sel].max()))
        if (~sel).any():
            lo_un = min(lo_un, int(z[~sel].min()))
    assert hi_sel < lo_un
    # spot check: a small prefix equals the oracle's draw restricted by that threshold
    assert np.array_equal(m[:1000], (MK.splitmix64_keys(seed, 1000) <= np.uint64(hi_sel)).astype(np.uint8))


def test_errors():
    from paper_2511_16358_b200 import IfctnError, _abi
    buf = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(IfctnError):
        _abi.ifctn_mask_uniform(buf.data_ptr(), 16, 17, 0)
    with pytest.raises(IfctnError):
        _abi.ifctn_mask_uniform(buf.data_ptr(), 16, -1, 0)
    host = np.zeros(16, np.uint8)
    with pytest.raises(IfctnError):
        _abi.ifctn_mask_uniform(host.ctypes.data, 16, 3, 0)
    with pytest.raises(IfctnError):
        _abi.ifctn_mask_fibres(buf.data_ptr(), (4, 4), 2, 1, 0)
    with pytest.raises(IfctnError):
        _abi.ifctn_mask_fibres(buf.data_ptr(), (4, 4), 0, 5, 0)


@pytest.mark.parametrize("kind", ["RM", "FM"])
def test_device_mask_drives_a_sweep(kind):
    """A device-drawn sampling set fed straight into ifctn_create: one sweep within the
    north-star 1e-4 of the oracle run on the oracle's own draw of the same set."""
    from oracle import oracle as O
    from paper_2511_16358_b200 import Solver, mask_fibres, mask_uniform
    from synth import make_problem

    from gpu_util import dev, rel
    p = make_problem("C4s-like", (14, 9, 12, 4), 3, np.float32, "normal", scale_noise=0.01, sr=0.1, sweeps=1)
    if kind == "RM":
        m_dev = mask_uniform(p.n, p.n // 10, 21)
        m = MK.mask_uniform(p.n, p.n // 10, 21)
    else:
        m_dev = mask_fibres(p.dims, 2, 300, 21)
        m = MK.mask_fibres(p.dims, 2, 300, 21)
    observed = np.where(m.astype(bool), p.truth, 0).astype(p.dtype)
    s = Solver(p.dims, p.ranks, dev(observed), m_dev, dev(p.G0), rho=p.rho)
    s.sweep(1)
    Xg = s.reconstruct().cpu().numpy()
    Gg = s.factors().cpu().numpy()
    s.close()
    sh = O.Shape(p.dims, p.ranks)
    G = p.G0.astype(np.float64)
    X = O.init_x(observed, m)
    st, _, _ = O.sweep(sh, G, X, m, p.rho, O.objective(sh, G, X), False)
    assert st == 0
    assert rel(Gg, G) <= 1e-4 and rel(Xg, X) <= 1e-4
    obs = m.astype(bool)
    assert np.array_equal(Xg[obs].view(np.uint8), observed[obs].view(np.uint8))


def test_select_fallback_passes():
    """The 8-bit fallback passes (taken when more keys than the candidate buffer share the
    24-bit prefix; forced here with IFCTN_MASK_CAND_CAP=0 in a child process) give the same
    draw."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from paper_2511_16358_b200 import mask_uniform, mask_fibres\n"
            "from oracle import masks as MK\n"
            "for n, k in [(1, 1), (17, 5), (100003, 31337)]:\n"
            "    assert np.array_equal(mask_uniform(n, k, 9).cpu().numpy(), MK.mask_uniform(n, k, 9))\n"
            "d = (7, 9, 11, 13)\n"
            "assert np.array_equal(mask_fibres(d, 1, 500, 4).cpu().numpy(), MK.mask_fibres(d, 1, 500, 4))\n"
            "print('ok')\n") % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IFCTN_MASK_CAND_CAP="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
