"""GPU: SDXL's text encoders (the step before the loop) on this
package's kernels vs the plain-torch fp32 restatement oracle/text_ref.py.
Parity is unpinned by the reference (no text encoders). Tolerance
for bf16 compute through a residual stack: max-abs error <= 5e-2 * max|ref|.
"""
import pytest
import torch

from oracle.text_ref import CLIPTextRef
from paper_2602_21760_b200.denoiser import kernels as K
from paper_2602_21760_b200.denoiser.text_encoders import (CLIP_TINY_A, CLIP_TINY_B, CLIPTextEncoder,
                                                          SDXLTextEncoders, clip_text_param_specs)
from paper_2602_21760_b200.denoiser.weights import init_weights

pytestmark = pytest.mark.gpu


def _ids(n, vocab, seq=77, seed=0):
    g = torch.Generator().manual_seed(seed)
    ids = torch.randint(1, vocab - 1, (n, seq), generator=g)
    for r in range(n):                                   # EOS (max id) at a per-row position
        ids[r, 5 + 7 * r:] = 0
        ids[r, 5 + 7 * r] = vocab - 1
    return ids.cuda()


def test_causal_attention_matches_torch():
    torch.manual_seed(0)
    B, H, S = 2, 3, 77
    qkv = torch.randn(B * S, 3 * H * 64, device="cuda").bfloat16()
    o = torch.empty(B * S, H * 64, device="cuda", dtype=torch.bfloat16)
    K.attention(qkv, qkv, qkv, o, batch=B, heads=H, sq=S, skv=S, scale=0.125, q_col0=0, k_col0=H * 64,
                v_col0=2 * H * 64, causal=True)
    q, k, v = qkv.float().view(B, S, 3, H, 64).permute(2, 0, 3, 1, 4)
    mask = torch.full((S, S), float("-inf"), device="cuda").triu(1)
    ref = (torch.softmax(q @ k.transpose(-1, -2) * 0.125 + mask, -1) @ v).transpose(1, 2).reshape(B * S, H * 64)
    assert (o.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item()


@pytest.mark.parametrize("spec", [CLIP_TINY_A, CLIP_TINY_B])
def test_clip_text_encoder_matches_fp32_reference(spec):
    W = init_weights(clip_text_param_specs(spec), seed=5, device="cuda")
    ids = _ids(2, spec.vocab)
    hid, pooled = CLIPTextEncoder(spec, W).encode(ids)
    rh, rp = CLIPTextRef(spec, W).encode(ids)
    assert hid.shape == rh.shape and pooled.shape == rp.shape
    assert (hid.float() - rh).abs().max().item() <= 5e-2 * rh.abs().max().item()
    assert (pooled - rp).abs().max().item() <= 5e-2 * rp.abs().max().item()


def test_sdxl_conditioning_shapes():
    wa = init_weights(clip_text_param_specs(CLIP_TINY_A), seed=1, device="cuda")
    wb = init_weights(clip_text_param_specs(CLIP_TINY_B), seed=2, device="cuda")
    enc = SDXLTextEncoders(CLIPTextEncoder(CLIP_TINY_A, wa), CLIPTextEncoder(CLIP_TINY_B, wb))
    cond = enc.conditioning(_ids(2, 1000), _ids(1, 1000, seed=9))
    assert cond.context.shape == (2, 77, 128 + 192) and cond.pooled.shape == (2, 128)
    assert cond.null_context.shape == (1, 77, 320) and cond.null_pooled.shape == (1, 128)
