"""Host-resident level features (the e2e serving path): sphinx_gather_halo_windows copies exactly the
halo windows of the listed blocks (from pinned host memory or from the device), and a step fed that
way computes bit for bit what the device-resident step computes."""
import numpy as np
import pytest

import oracle
import synthetic as syn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
dev = "cuda"


def _window_mask(ids, n, h, b):
    hb = -(-h // b)
    m = np.zeros((n, h, h), bool)
    for i in ids:
        f, r = divmod(int(i), hb * hb)
        by, bx = divmod(r, hb)
        m[f, max(by * b - 1, 0):min(by * b + b + 1, h), max(bx * b - 1, 0):min(bx * b + b + 1, h)] = True
    return m


@pytest.mark.parametrize("geom", [(3, 72, 320), (2, 36, 640), (4, 18, 1280), (2, 20, 64)])
@pytest.mark.parametrize("pinned", [True, False])
def test_gather_halo_windows(sphinx, geom, pinned):
    n, h, c = geom
    b = 8
    hb = -(-h // b)
    rg = np.random.default_rng(h * c + pinned)
    m = (rg.random((n, hb, hb)) < 0.3).astype(np.uint8)
    ids_np = np.flatnonzero(m.ravel()).astype(np.int32)
    ids = torch.from_numpy(ids_np).to(dev)
    cnt = torch.tensor([len(ids_np)], dtype=torch.int32, device=dev)
    bits = syn.features_bf16((n, h, h, c), f"hw{h}")
    src = torch.from_numpy(bits.view(np.int16))
    src = src.pin_memory() if pinned else src.to(dev)
    dst = torch.full((n, h, h, c), 0x7F7F, dtype=torch.int16, device=dev)
    sphinx.sphinx_gather_halo_windows(src.view(torch.bfloat16), dst.view(torch.bfloat16), b, ids, cnt)
    torch.cuda.synchronize()
    got = dst.cpu().numpy()
    win = _window_mask(ids_np, n, h, b)
    assert np.array_equal(got[win], bits.view(np.int16)[win])
    assert np.all(got[~win] == 0x7F7F)


def test_step_with_host_features_bitwise(sphinx):
    from paper_2511_18672_b200.step import RefinementStep, StepConfig
    cfg = StepConfig(frames_per_request=6, n_requests=2)
    batch = syn.make_batch([0.3, 0.6], tag="hostfeat", frames_per_request=cfg.frames_per_request)
    d = torch.device(dev)
    ref = RefinementStep(cfg, batch, d, sphinx)
    hfeat = {l: torch.from_numpy(np.ascontiguousarray(batch[f"feat{l}"]).view(np.int16)).pin_memory()
             .view(torch.bfloat16) for l in range(cfg.L)}
    st = RefinementStep(cfg, batch, d, sphinx, host_features=hfeat)
    for l in range(cfg.L):  # the device maps start from garbage: only the gathered windows may matter
        st.d[f"feat{l}"].view(torch.int16).fill_(0x7FC0)
    ref.run()
    st.run()
    torch.cuda.synchronize()
    for l in range(cfg.L):
        assert torch.equal(ref.out(l).view(torch.int16), st.out(l).view(torch.int16)), l
    assert torch.equal(ref.lat_out, st.lat_out)
    assert st.window_bytes() > 0
