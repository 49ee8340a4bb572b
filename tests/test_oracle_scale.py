"""Pin the CPU oracle at the BASELINE scales: its outputs at configs C2 (500k,
1280x720), the north-star (2M, 1280x720), C3 (2M, 1297x840, with
render_backward) and C5 (5M, 1920x1080, sigma=0.1) must match the digests the
live reference produced (tests/golden/make_golden_scale.py).  The GPU parity
tests at these sizes then compare the CUDA path with this pinned oracle."""
import numpy as np
import pytest

import scale_golden as SG


def _oracle_forward(name):
    from oracle import oracle as O
    from paper_2505_19175_b200 import scenes
    z = SG.load(name)
    soup, intr, pose = scenes.make_scene(name)
    SG.check_inputs(z, soup)
    ref = O.render(soup, intr, pose)
    SG.check_forward(z, sorted_idx=ref.proj.sorted_idx, tile_start=ref.tile_start, entry_tri=ref.entry_tri,
                     last_src=ref.last_src, nfrag=ref.nfrag, pixcount=ref.per_triangle_pixel_count,
                     image=ref.image, alpha=ref.alpha_map, maxw=ref.per_triangle_max_weight,
                     area=ref.per_triangle_area, label=f"oracle-{name}")
    return z, soup, intr, pose


@pytest.mark.parametrize("name", ["c2", "ns", "c5"])
def test_oracle_forward_matches_reference_at_scale(name):
    _oracle_forward(name)


def test_oracle_backward_matches_reference_at_c3():
    from oracle import oracle as O
    from paper_2505_19175_b200 import scenes
    from conftest import digest
    z, soup, intr, pose = _oracle_forward("c3")
    d_image = scenes.make_d_image(3, intr.height, intr.width, fp32=True)
    assert digest(d_image) == str(z["d_image_digest"])
    g = O.render_backward(soup, intr, pose, d_image=d_image)
    rows = SG.grad_rows(g)
    # the oracle is fp64 like the reference: far inside the gradient tolerance
    nb, worst = SG.grad_violations(rows[z["tri_sample"]], z["grad_sample"], rtol=1e-9, atol=1e-12)
    assert nb == 0, f"{nb} sampled gradients differ (worst {worst})"
    SG.check_grad_sample(z, rows, "oracle-c3")
