"""fp8 wire for the cross-node dispatch legs (moe_ctx_set_wire, SURVEY.md
§8(f) item 3): every landed row that crossed a node equals the e4m3 round
trip of its source row — per 128-element block, scale = amax / 448 (fp32),
q = e4m3_rn_satfinite(x / scale), row = bf16(q * scale) — bit for bit (an
emulation of the wire format in PyTorch); own-node rows stay bit-exact; the
layer output (the combine's reverse AllToAll on the same wire: crossed slots
make a second round trip) stays within the combine bound of those rows."""
import numpy as np
import pytest
import torch

import oracle
from paper_2411_00662_b200 import _lib
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED

pytestmark = pytest.mark.gpu


def _fp8_roundtrip(rows: torch.Tensor) -> torch.Tensor:
    """bf16 [n, h] -> the wire's decode of its encode (blocks of 128 columns)."""
    n, h = rows.shape
    f = rows.float().view(n, h // 128, 128)
    amax = f.abs().amax(-1, keepdim=True)
    scale = torch.where(amax > 0, amax / 448.0, torch.ones_like(amax))
    q = (f / scale).clamp(-448.0, 448.0).to(torch.float8_e4m3fn).float()
    return (q * scale).view(n, h).to(torch.bfloat16)


@pytest.mark.parametrize("e,t,E,k,level,n", [(2, 2, 8, 2, O1, 1), (2, 1, 8, 2, BASELINE, 1), (4, 2, 16, 4, O1, 1),
                                             (2, 2, 8, 2, O2, 4), (2, 2, 8, 2, O3, 2), (2, 2, 8, 2, BASELINE, 1)])
def test_fp8_wire_rows_and_combine(cuda, e, t, E, k, level, n):
    T, h = 256, 512
    g = torch.Generator().manual_seed(e * 100 + t * 10 + level + n)
    x = (torch.randn(e, T, h, generator=g) * torch.logspace(-3, 3, h)[None, None, :]).to(torch.bfloat16)
    logits = torch.randn(e, T, E, generator=g)
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=max(n, 1))
    try:
        layer.set_wire(_lib.WIRE_FP8)
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
        layer.route()
        layer.dispatch(level, n, LAND_FINAL)
        layer.sync()
        experts = np.stack([layer.card(gg * t).experts.cpu().numpy() for gg in range(e)])
        nodes = oracle.Nodes(e, t, E, x.contiguous().view(torch.uint8).numpy().reshape(e, T, -1), experts)
        fin = nodes.dispatch_monolithic()
        rt = torch.stack([_fp8_roundtrip(x[gg]) for gg in range(e)])  # [e, T, h]
        for cd in layer.cards:
            rows = layer.recv_rows(cd.card)
            want_rows, want_tags = fin[cd.node]
            assert rows == want_rows.shape[0]
            np.testing.assert_array_equal(cd.recv_tags[:rows].cpu().numpy(), want_tags)
            got = cd.recv[:rows].cpu()
            src = torch.from_numpy(want_tags[:, 1] // t).long()
            pos = torch.from_numpy(want_tags[:, 2]).long()
            own = src == cd.node
            want = torch.from_numpy(want_rows.copy()).view(torch.bfloat16).reshape(rows, h).clone()
            want[~own] = rt[src[~own], pos[~own]]  # crossed a node: the fp8 round trip
            assert torch.equal(got.view(torch.int16), want.view(torch.int16)), cd.card
            if (~own).any():  # and that round trip is lossy but bounded: one e4m3 rounding
                xs = x[src[~own], pos[~own]].float()
                scale = xs.view(-1, h // 128, 128).abs().amax(-1, keepdim=True).expand(-1, -1, 128).reshape(xs.shape) / 448
                bound = (2.0 ** -4 + 2.0 ** -8) * xs.abs() + scale * 2.0 ** -9
                assert ((got[~own].float() - xs).abs() <= bound).all()
        layer.combine(level, n)
        layer.sync()
        # the combine's reverse AllToAll is on the fp8 wire too: a crossed slot's
        # expert output (here the dispatched row itself) makes a second round trip
        rt2 = torch.stack([_fp8_roundtrip(rt[gg]) for gg in range(e)])
        for cd in layer.cards:
            ex = torch.from_numpy(experts[cd.node]).long()
            pr = cd.probs.float().cpu()
            L = E // e
            ref = torch.zeros(T, h)
            for s in range(k):
                crossed = (ex[:, s] // L) != cd.node
                row = torch.where(crossed[:, None], rt2[cd.node].float(), x[cd.node].float())
                ref += pr[:, s:s + 1] * row
            got = cd.out.float().cpu()
            assert ((got - ref).abs() <= 2.0 ** -8 * ref.abs() + 1e-6 * ref.abs().amax()).all(), cd.card
    finally:
        layer.close()


def test_fp8_wire_validation(cuda):
    layer = MoeLayer(2, 2, 8, 2, 64, 192, dtype=torch.bfloat16, max_chunks=2)
    try:
        with pytest.raises(ValueError):
            layer.set_wire(_lib.WIRE_FP8)  # hidden/t = 96 is not a multiple of 128
    finally:
        layer.close()
    layer = MoeLayer(2, 2, 8, 2, 64, 256, dtype=torch.bfloat16, max_chunks=2)
    try:
        layer.set_wire(_lib.WIRE_FP8)
        with pytest.raises(ValueError):
            layer.dispatch(O2, 2, LAND_STAGED)  # the fp8 wire lands in pre
        layer.set_wire(_lib.WIRE_BF16)
        layer.route()
        layer.dispatch(O2, 2, LAND_STAGED)
        layer.sync()
    finally:
        layer.close()
