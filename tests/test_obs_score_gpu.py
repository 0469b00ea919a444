"""K5 (tcgen05 observation-window scoring) vs the fp32 oracle.

window = 1 is the reference's step-0 semantics (last prompt token, GQA mean,
export.ts:125-127 / model.ts:274-291); window > 1 averages the causal
softmax rows of the last `window` prompt tokens.  Tolerance: 2e-6 absolute
+ 2e-3 relative on the probability rows (bf16 inputs, fp32 accumulation in
TMEM, exp2 on the GPU).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _oracle_rows(k, q, B, H, G, w, L):
    import torch

    out = np.zeros((B * H, L), dtype=np.float64)
    for b in range(B):
        for h in range(H):
            kk = k[b * H + h].double()
            acc = torch.zeros(L, dtype=torch.float64)
            for i in range(w):
                lim = L - w + i  # query position, sees keys <= lim
                for j in range(G):
                    s = (q[b, i, h * G + j].double() @ kk[:lim + 1].T) / math.sqrt(128)
                    acc[:lim + 1] += torch.softmax(s, -1)
            out[b * H + h] = (acc / (w * G)).numpy()
    return out


@pytest.mark.parametrize("B,H,G,w,L", [(1, 2, 4, 1, 700), (2, 2, 7, 1, 1300), (1, 2, 4, 32, 1000),
                                       (1, 1, 8, 16, 9000), (2, 3, 4, 5, 4097),
                                       # w*G <= 16: K read once, probabilities from kept scores
                                       (2, 2, 4, 4, 3001), (1, 2, 8, 2, 777), (1, 3, 1, 1, 50)])
def test_obs_scores_match_oracle(B, H, G, w, L):
    import torch

    from paper_2601_13684_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(L + w)
    k = torch.randn(B * H, L, 128, device="cuda", generator=g).to(torch.bfloat16)
    q = (torch.randn(B, w, H * G, 128, device="cuda", generator=g) * 2).to(torch.bfloat16)
    stride = (L + 3) // 4 * 4
    rows = torch.zeros(B * H, stride, device="cuda")
    _lib.check(_lib.load().hc_obs_scores(k.data_ptr(), q.data_ptr(), B, H, G, w, L,
                                         rows.data_ptr(), stride, _lib.stream_handle()))
    torch.cuda.synchronize()
    got = rows[:, :L].cpu().numpy()
    exp = _oracle_rows(k.float().cpu(), q.float().cpu(), B, H, G, w, L)
    assert np.allclose(got, exp, atol=2e-6, rtol=2e-3), float(np.abs(got - exp).max())
    assert np.allclose(got.sum(1), 1.0, atol=1e-3)  # each row is a probability mean
