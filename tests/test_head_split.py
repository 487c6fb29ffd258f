"""Pin of the head's operand split (net_layers.cu fc_kernel, DESIGN.md kernel table):
the classifier runs bf16 tensor-core MMAs on p = p0 + p1 + p2, each term the RNE bf16 of
the remainder of an fp32 pooled feature, and claims the split is EXACT (3 x 8
significand bits cover fp32's 24, and bf16 shares fp32's exponent range), so the three
MMAs over the same bf16 weights see the fp32 operand.  Precisely: exact whenever |p| >= 2^-110
(the third term's lowest bit, 2^(e-23), is then >= bf16's smallest subnormal 2^-133); below that
the split's absolute error is < 2^-133.  Checked here with torch's RNE casts on random,
extreme and boundary fp32 values."""
import numpy as np
import torch


def _split3(p: torch.Tensor):
    p0 = p.to(torch.bfloat16).float()
    r1 = p - p0
    p1 = r1.to(torch.bfloat16).float()
    r2 = r1 - p1
    p2 = r2.to(torch.bfloat16).float()
    return p0, p1, p2, r2


def test_three_term_bf16_split_is_exact():
    g = torch.Generator().manual_seed(11)
    vals = [torch.randn(1 << 20, generator=g),
            torch.randn(1 << 18, generator=g) * 1e-30,
            torch.randn(1 << 18, generator=g) * 1e30,
            torch.rand(1 << 18, generator=g) * 8.0]
    bits = torch.randint(0, 1 << 31, (1 << 20,), generator=g, dtype=torch.int64).to(torch.int32)
    raw = bits.view(torch.float32)
    vals.append(raw[torch.isfinite(raw) & (raw.abs() < 1e37)])  # random bit patterns (incl. subnormals)
    edge = np.array([1.0 + 2.0 ** -23, 1.0 - 2.0 ** -24, 3.0 - 2.0 ** -22, 2.0 ** -126, 2.0 ** -149,
                     65504.0, 1.0 / 3.0, -2.0 / 3.0, 0.0], dtype=np.float32)
    vals.append(torch.from_numpy(edge))
    for p in vals:
        p0, p1, p2, r2 = _split3(p)
        total = p0.double() + p1.double() + p2.double()
        big = (p.abs() >= 2.0 ** -110) | (p == 0)
        assert big.any()
        assert torch.equal(r2[big], p2[big]), "the third term must be exact in bf16"
        assert torch.equal(total[big], p.double()[big]), "p0 + p1 + p2 == p"
        assert float((total - p.double()).abs().max()) < 2.0 ** -133  # tiny values: below bf16's subnormal step
