"""Host-side helpers of the C5 encoder (no GPU needed)."""
import pytest


def test_encoder_precision_helpers():
    import torch

    from paper_2603_00035_b200 import training

    assert training.ENCODER_PRECISIONS == ("fp32", "bf16")
    m = training.prepare_encoder(training.RandersEncoder(), "bf16")
    assert m.convs[1].weight.is_contiguous(memory_format=torch.channels_last)
    x = training.encoder_input(torch.zeros(2, 3, 8, 8), "bf16")
    assert x.is_contiguous(memory_format=torch.channels_last)
    assert training.encoder_input(x, "fp32") is x
    with pytest.raises(ValueError):
        training.encoder_autocast("fp16")
