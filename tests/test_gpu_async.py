"""Asynchronous forwards (ts_set_async): an entry-capacity overflow of a frame
that nobody polls is reported by the next forward (it used to render
background silently until ts_forward_status), the status call grows the
capacity, and the repeated frame matches a synchronous one."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_async_overflow_is_reported_by_the_next_forward():
    from paper_2505_19175_b200 import scenes
    from paper_2505_19175_b200.rasterizer import DeviceSoup, Rasterizer
    r = Rasterizer()
    intr, pose = scenes.frontal_camera(256, 192, 300.0)
    sparse = DeviceSoup.from_soup(scenes.make_soup(2000, seed=1, size=0.05, sigma=1.0), dtype=torch.float32)
    dense = DeviceSoup.from_soup(scenes.make_soup(60000, seed=2, size=0.3, sigma=1.0), dtype=torch.float32)
    ref = r.forward(dense, intr, pose, keep_backward=False)  # synchronous: grows as needed
    img_ref = ref.image.clone()
    r2 = Rasterizer()
    r2.forward(sparse, intr, pose, keep_backward=False)       # small working capacity
    r2.set_async(True)
    r2.forward(dense, intr, pose, keep_backward=False)        # outgrows it
    torch.cuda.synchronize()
    with pytest.raises(RuntimeError, match="capacity"):
        r2.forward(dense, intr, pose, keep_backward=False)
    with pytest.raises(RuntimeError, match="capacity"):
        r2.status()                                           # clears the flag, grows the capacity
    f = r2.forward(dense, intr, pose, keep_backward=False)
    r2.status()
    r2.set_async(False)
    assert np.array_equal(f.image.cpu().numpy(), img_ref.cpu().numpy())


def test_concurrent_contexts_on_streams():
    """Frames in flight on three contexts, one stream each (bench.py
    concurrent_frames): every frame equals the single-context frame."""
    from paper_2505_19175_b200 import DeviceSoup, Rasterizer, scenes
    soup = DeviceSoup.from_soup(scenes.make_soup(50_000, seed=3, size=0.05, sigma=(1.0, 1.0)), dtype=torch.float32)
    intr, pose = scenes.frontal_camera(320, 240, 300.0)
    poses = scenes.orbit_cameras(6, seed=4)
    ref = Rasterizer()
    want = [ref.forward(soup, intr, p, keep_backward=False).image.clone() for p in poses]
    rs = [Rasterizer() for _ in range(3)]
    sts = [torch.cuda.Stream() for _ in range(3)]
    for r, st in zip(rs, sts):  # (sizes the buffers), then asynchronous frames in flight
        with torch.cuda.stream(st):
            r.forward(soup, intr, poses[0], keep_backward=False)
        r.set_async(True)
    torch.cuda.synchronize()
    outs = []
    for i, p in enumerate(poses):
        with torch.cuda.stream(sts[i % 3]):
            outs.append(rs[i % 3].forward(soup, intr, p, keep_backward=False).image)
    torch.cuda.synchronize()
    for r, st in zip(rs, sts):
        r.status(stream=st)
        r.set_async(False)
    for got, w in zip(outs, want):
        assert torch.equal(got, w)


def test_forward_captured_in_cuda_graph():
    """An asynchronous forward captured in a CUDA graph (stream capture of the
    whole frame: counter reset, preprocess, binning, sort, blend, fix-up) replays
    to the eager frame; the same soup buffers updated in place render anew."""
    from paper_2505_19175_b200 import DeviceSoup, Rasterizer, scenes
    soup = DeviceSoup.from_soup(scenes.make_soup(50_000, seed=3, size=0.05, sigma=(1.0, 1.0)), dtype=torch.float32)
    intr, pose = scenes.frontal_camera(320, 240, 300.0)
    r = Rasterizer()
    want = r.forward(soup, intr, pose, keep_backward=False).image.clone()
    r.set_async(True)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            r.forward(soup, intr, pose, keep_backward=False)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = r.forward(soup, intr, pose, keep_backward=False)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.image, want)
    # parameters changed in place: the replay renders the new values
    soup.sh.mul_(0.5)
    g.replay()
    torch.cuda.synchronize()
    r.status()
    r.set_async(False)
    want2 = Rasterizer().forward(soup, intr, pose, keep_backward=False).image
    assert torch.equal(out.image, want2) and not torch.equal(want2, want)
