"""GPU: fused cross-entropy (loss + bf16 dlogits, csrc/train_ops.cu) against a
plain PyTorch fp32 reference, on the vectorised path (vocab % 8 == 0, the
50304-word head) and the scalar path (ragged vocab).  Tolerances: loss 1e-5
relative (fp32 sums in a different order), dlogits within bf16 rounding."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows,vocab", [(64, 50304), (7, 517), (3, 8), (33, 4096)])
def test_cross_entropy_matches_torch(cuda, rows, vocab):
    import torch
    from paper_2301_11913_b200 import _lib as L
    g = torch.Generator(device="cuda").manual_seed(rows * vocab)
    logits = torch.randn(rows, vocab, device="cuda", generator=g) * 4
    targets = torch.randint(0, vocab, (rows,), device="cuda", generator=g, dtype=torch.int32)
    targets[0] = vocab - 1
    targets[-1] = 0
    loss = torch.zeros(1, device="cuda")
    dl = torch.empty(rows, vocab, dtype=torch.bfloat16, device="cuda")
    scale = 1.0 / rows
    rc = L.lib().swarm_cross_entropy(logits.data_ptr(), targets.data_ptr(), rows, vocab, scale, loss.data_ptr(),
                                     dl.data_ptr(), torch.cuda.current_stream().cuda_stream)
    L.check(rc, "cross_entropy")
    torch.cuda.synchronize()
    ref_loss = torch.nn.functional.cross_entropy(logits, targets.long(), reduction="sum")
    assert abs(loss.item() - ref_loss.item()) <= 1e-5 * abs(ref_loss.item()) + 1e-4
    p = torch.softmax(logits, dim=1)
    p[torch.arange(rows), targets.long()] -= 1.0
    ref_d = p * scale
    err = (dl.float() - ref_d).abs()
    assert float(err.max()) <= float(ref_d.abs().max()) * 2 ** -7 + 1e-7
