"""The asynchronous device API: data-dependent decisions are taken on the device.

The soft-mask range check, the f32 / f64 choice for lambda = 1 and GSF's
empty-complement skip set a gate word that the transform's kernels test, so a
GD_MEM_DEVICE call enqueues everything and returns without blocking; errors
found on the device are deferred to the next call / gd_synchronize (the
reference validates before computing: transforms.cpp:22-28, 143-158, 204-219)."""
import time

import numpy as np
import pytest

from tests.helpers import bitwise_equal, dyadic_image, parity, point_mask

pytestmark = pytest.mark.gpu


@pytest.fixture
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def test_device_call_returns_before_the_gpu_finishes(gd, torch_cuda):
    torch = torch_cuda
    shape = (256, 256, 256)
    img = torch.empty(shape, device="cuda")
    gd.device.fill_splitmix(img, 7)
    mask = torch.ones(shape, device="cuda")
    mask[128, 128, 128] = 0.0
    out = torch.empty_like(img)
    for _ in range(2):
        gd.device.generalized_geodesic(img, mask, out, None, 1.0, 1e10, 4)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    gd.device.generalized_geodesic(img, mask, out, None, 1.0, 1e10, 4)
    host_ms = (time.perf_counter() - t0) * 1e3
    b.record()
    torch.cuda.synchronize()
    gpu_ms = a.elapsed_time(b)
    assert host_ms < gpu_ms / 2, (host_ms, gpu_ms)  # no host synchronisation inside the call
    gd.device.synchronize()


def test_bad_mask_is_a_deferred_error(gd, torch_cuda):
    torch = torch_cuda
    shape = (8, 16, 20)
    img = torch.zeros(shape, device="cuda")
    mask = torch.full(shape, 2.0, device="cuda")
    out = torch.empty_like(img)
    gd.device.generalized_geodesic(img, mask, out, None, 1.0, 1e10, 2)  # enqueued, no error yet
    with pytest.raises(gd.InvalidArgument):
        gd.device.synchronize()
    gd.device.synchronize()  # reported once
    mask.fill_(1.0)
    mask[4, 8, 10] = 0.0
    gd.device.generalized_geodesic(img, mask, out, None, 1.0, 1e10, 2)
    gd.device.synchronize()
    # host-memory calls report it synchronously and leave the output untouched
    with pytest.raises(gd.InvalidArgument):
        gd.generalized_geodesic(np.zeros(shape, np.float32), np.full(shape, -1.0, np.float32))


def test_lambda1_f32_or_f64_chosen_on_the_device(gd, oracle, torch_cuda):
    """Dyadic image: the f32 sweeps run, the f64 twins leave at once; a
    many-binade image: the reverse.  Both bit-exact against the oracle."""
    torch = torch_cuda
    shape = (16, 33, 40)
    rng = np.random.default_rng(5)
    m = point_mask(shape)
    for name, img in (("dyadic", dyadic_image(rng, shape)),
                      ("binades", (rng.standard_normal(shape) * 1000).astype(np.float32))):
        d_img = torch.from_numpy(img).cuda()
        d_m = torch.from_numpy(m).cuda()
        out = torch.empty_like(d_img)
        gd.launch_log(reset=True)
        gd.device.generalized_geodesic(d_img, d_m, out, None, 1.0, 1e10, 2)
        gd.device.synchronize()
        log = gd.launch_log(reset=True)
        assert {r["f64"] for r in log} == {0, 1}, name  # both enqueued, the gate picks one
        want = oracle.generalized_geodesic(img, m, None, 1.0, 1e10, 2)
        assert bitwise_equal(out.cpu().numpy(), want), (name, parity(out.cpu().numpy(), want))


def test_gsf_complement_skip_on_device(gd, oracle, torch_cuda):
    torch = torch_cuda
    img = torch.zeros((1, 5), device="cuda")
    mask = torch.tensor([[1, 1, 0, 1, 1]], dtype=torch.float32, device="cuda")
    out = torch.empty_like(img)
    st = gd.device.gsf(img, mask, out, None, 0.0, 1e10, 2, 1.0)  # stats requested: synchronises
    assert st.complement_empty == 1 and st.rounds == 2
    assert torch.all(out == 1.0)
    # the reference's general case, with and without the erode
    shape = (12, 20, 18)
    rng = np.random.default_rng(9)
    h_img = dyadic_image(rng, shape)
    h_mask = (rng.random(shape) < 0.5).astype(np.float32)
    for theta in (0.0, 2.0, 50.0):
        d_out = torch.empty((shape), device="cuda")
        st = gd.device.gsf(torch.from_numpy(h_img).cuda(), torch.from_numpy(h_mask).cuda(), d_out,
                           None, 1.0, 1e10, 2, theta)
        want, rounds, ce = oracle.gsf(h_img, h_mask, None, 1.0, 1e10, 2, theta)
        assert bitwise_equal(d_out.cpu().numpy(), want), theta
        assert (st.rounds, bool(st.complement_empty)) == (rounds, ce), theta


def test_batched_host_pipeline(gd, oracle):
    """Host-memory batches run pipelined in chunks (H2D / transform / D2H on three
    streams): every volume still matches the oracle, and a bad mask in a later
    chunk is reported."""
    rng = np.random.default_rng(17)
    B, shape = 13, (20, 64, 72)
    imgs = dyadic_image(rng, (B,) + shape)
    masks = np.ones((B,) + shape, np.float32)
    for b in range(B):
        masks[b].reshape(-1)[rng.integers(0, masks[b].size)] = 0.0
    g = gd.generalized_geodesic_batched(imgs, masks, (1.0, 1.0, 2.5), 1.0, 1e10, 2)
    for b in (0, 6, 12):
        want = oracle.generalized_geodesic(imgs[b], masks[b], (1.0, 1.0, 2.5), 1.0, 1e10, 2)
        assert bitwise_equal(g[b], want), b
    masks[11, 0, 0, 0] = 3.0
    with pytest.raises(gd.InvalidArgument):
        gd.generalized_geodesic_batched(imgs, masks, (1.0, 1.0, 2.5), 1.0, 1e10, 2)
    masks[11, 0, 0, 0] = 1.0
    gd.generalized_geodesic_batched(imgs, masks, (1.0, 1.0, 2.5), 1.0, 1e10, 2)


def test_concurrent_streams_are_independent(gd, torch_cuda):
    """Transforms enqueued on several CUDA streams at once (each stream has its own
    workspace, halo words and gate) give exactly the single-stream results."""
    torch = torch_cuda
    shape, B, ns = (24, 40, 96), 12, 3
    img = torch.empty((B,) + shape, device="cuda")
    for b in range(B):
        gd.device.fill_splitmix(img[b], 300 + b)
    mask = torch.ones_like(img)
    mask[:, 12, 20, 48] = 0.0
    want = {}
    for lam in (0.0, 0.6, 1.0):
        ref = torch.empty_like(img)
        gd.device.generalized_geodesic(img, mask, ref, (1.0, 1.0, 2.5), lam, 1e10, 3, batch=B)
        want[lam] = ref
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(ns)]
    outs = {lam: torch.full_like(img, -1.0) for lam in want}
    per = B // ns
    for lam in want:  # every stream busy with every lambda, interleaved
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                sl = slice(i * per, (i + 1) * per)
                gd.device.generalized_geodesic(img[sl], mask[sl], outs[lam][sl], (1.0, 1.0, 2.5),
                                               lam, 1e10, 3, batch=per, stream=s.cuda_stream)
    for s in streams:
        cur.wait_stream(s)
    torch.cuda.synchronize()
    gd.device.synchronize()
    for lam in want:
        assert torch.equal(outs[lam].view(torch.int32), want[lam].view(torch.int32)), lam
