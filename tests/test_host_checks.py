"""Host-side argument checks that run before any device work (CPU)."""
import pytest
import torch

from paper_2512_02932_b200 import raster
from paper_2512_02932_b200.errors import ConfigError


def _outs(h, w, dev="cpu"):
    return dict(color=torch.empty((h, w, 3), device=dev), depth=torch.empty((h, w), device=dev),
                transmittance=torch.empty((h, w), device=dev), alpha=torch.empty((h, w), device=dev),
                normal=torch.empty((h, w, 3), device=dev))


def test_output_buffers_of_the_camera_shape_pass():
    raster._check_outputs(_outs(6, 8), 6, 8, torch.device("cpu"))
    raster._check_outputs({"color": None}, 6, 8, torch.device("cpu"))


@pytest.mark.parametrize("bad", ["shape", "dtype", "strided", "name", "device"])
def test_output_buffers_that_would_be_overrun_are_rejected(bad):
    o = _outs(6, 8)
    dev = torch.device("cpu")
    if bad == "shape":
        o["depth"] = torch.empty((6, 9))
    elif bad == "dtype":
        o["color"] = torch.empty((6, 8, 3), dtype=torch.float64)
    elif bad == "strided":
        o["normal"] = torch.empty((6, 8, 6))[:, :, ::2]
    elif bad == "name":
        o["colour"] = torch.empty((6, 8, 3))
    else:
        dev = torch.device("meta")
    with pytest.raises(ConfigError):
        raster._check_outputs(o, 6, 8, dev)
