"""Small batches with the default dispatch (the conftest lifts the K3p / K3c small-batch
thresholds for the other tests): DCGAN layers at batch 1 and 4 route to K3 with narrow N tiles
and split K (csrc/igemm_sm100.cu make_params), larger batches to K3p / K3c, and every one of them
matches the oracle at the bf16 gate (fp32 output on bf16-rounded operands: rel 1e-4 / abs 1e-5,
DESIGN.md section 4)."""
import numpy as np
import pytest

import paper_2502_20493_b200 as P
from oracle import segconv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture()
def defaults(monkeypatch):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    monkeypatch.delenv("SEGB200_K3P_MIN_TILES", raising=False)
    monkeypatch.delenv("SEGB200_K3C_MIN_TILES", raising=False)
    return torch


@pytest.mark.parametrize("name,h,ci,co,batch,family", [
    ("dcgan_l2", 4, 1024, 512, 1, "K3 "), ("dcgan_l3", 8, 512, 256, 1, "K3 "),
    ("dcgan_l4", 16, 256, 128, 1, "K3 "), ("dcgan_l4", 16, 256, 128, 4, "K3 "),
    ("dcgan_l4", 16, 256, 128, 64, "K3p"), ("dcgan_l5", 32, 128, 3, 1, "K3 "),
    ("dcgan_l5", 32, 128, 3, 16, "K3c"),
])
def test_small_batch_dispatch_and_parity(defaults, name, h, ci, co, batch, family):
    torch = defaults
    bank = O.gen_kernel_bank(ci, co, 4, 3)
    layer = P.prepare_layer(bank, 2, compute="bf16")
    assert layer.describe_path(batch, h, h).startswith(family), layer.describe_path(batch, h, h)
    x = torch.from_numpy(O.unit_floats(batch * ci * h * h, 9).reshape(batch, ci, h, h)).cuda().to(torch.bfloat16)
    y = layer.forward(x, out_dtype=torch.float32).cpu().numpy()
    ref = O.forward_segregated_batch(x.float().cpu().numpy().astype(np.float64),
                                     O.bf16_round(bank).astype(np.float64), 2)
    assert O.compare(y, ref, 1e-4, 1e-5)["passed"]
