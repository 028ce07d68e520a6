"""BatchNorm folding used by the EE inference benches (ee_infer.fold_batchnorm):
the folded ResNet computes the same function as the eval-mode original."""
import pytest
import torch

torchvision = pytest.importorskip("torchvision")

from paper_2312_05385_b200 import ee_infer


@pytest.mark.parametrize("ctor", [torchvision.models.resnet18, torchvision.models.resnet50])
def test_fold_batchnorm_preserves_eval_forward(ctor):
    torch.manual_seed(0)
    m = ctor().eval()
    for mod in m.modules():  # non-trivial statistics
        if isinstance(mod, torch.nn.BatchNorm2d):
            mod.running_mean.uniform_(-0.5, 0.5)
            mod.running_var.uniform_(0.5, 2.0)
            mod.weight.data.uniform_(0.5, 1.5)
            mod.bias.data.uniform_(-0.2, 0.2)
    x = torch.randn(2, 3, 64, 64)
    with torch.no_grad():
        ref = m(x)
        ee_infer.fold_batchnorm(m)
        got = m(x)
    assert torch.allclose(got, ref, rtol=1e-4, atol=1e-4 * ref.abs().max().item())
