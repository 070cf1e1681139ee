import pytest
import torch


@pytest.fixture(autouse=True, scope="session")
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device", allow_module_level=True)
    torch.cuda.set_device(0)
