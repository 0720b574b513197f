"""GPU: the VAE decoder (the step after the loop) on this
package's kernels vs the plain-torch fp32 restatement oracle/vae_ref.py with
the same random-init weights. Parity is unpinned by the reference (it has no
decoder); tolerance as for the U-Net (bf16 compute): max-abs error
<= 5e-2 * max|ref|, mean-abs error <= 1e-2 * mean|ref|.
"""
import pytest
import torch

from oracle.vae_ref import VAEDecoderRef
from paper_2602_21760_b200.denoiser import kernels as K
from paper_2602_21760_b200.denoiser.vae import VAEDecoder, vae_decoder_flops
from paper_2602_21760_b200.denoiser.weights import VAE_TINY, init_weights, vae_decoder_param_specs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny():
    return init_weights(vae_decoder_param_specs(VAE_TINY), seed=3, device="cuda")


def test_softmax_rows_matches_torch():
    torch.manual_seed(0)
    for rows, cols in [(7, 256), (300, 4096), (3, 16384)]:
        x = (torch.randn(rows, cols, device="cuda") * 4).bfloat16()
        y = K.softmax_rows(x, scale=0.3)
        ref = torch.softmax(x.float() * 0.3, dim=-1)
        assert (y.float() - ref).abs().max().item() <= 1e-2 * ref.max().item()
        assert torch.allclose(y.float().sum(-1), torch.ones(rows, device="cuda"), atol=2e-2)


@pytest.mark.parametrize("n", [1, 2])
def test_vae_decoder_matches_fp32_reference(tiny, n):
    torch.manual_seed(n)
    z = torch.randn(n, VAE_TINY.latent_hw, VAE_TINY.latent_hw, 4, device="cuda") * 0.5
    img = VAEDecoder(VAE_TINY, tiny).decode(z)
    ref = VAEDecoderRef(VAE_TINY, tiny).decode(z)
    assert img.shape == (n, 8 * VAE_TINY.latent_hw, 8 * VAE_TINY.latent_hw, 3) == ref.shape
    err = (img - ref).abs()
    assert err.max().item() <= 5e-2 * ref.abs().max().item()
    assert err.mean().item() <= 1e-2 * ref.abs().mean().item()


def test_vae_flops_positive():
    assert vae_decoder_flops(VAE_TINY, 1) > 0


def test_decode_latents_from_a_run_result(tiny):
    """x0 as the loop returns it (flat [B, h*w*4] NHWC, numpy) -> images."""
    import numpy as np
    from paper_2602_21760_b200 import pipelines
    vae = VAEDecoder(VAE_TINY, tiny)
    x0 = np.random.default_rng(0).standard_normal((2, VAE_TINY.latent_hw * VAE_TINY.latent_hw * 4)) * 0.5
    img = pipelines.decode_latents(vae, x0, VAE_TINY.latent_hw)
    ref = VAEDecoderRef(VAE_TINY, tiny).decode(torch.as_tensor(x0).reshape(2, 16, 16, 4).cuda())
    assert img.shape == (2, 128, 128, 3)
    assert (img - ref).abs().max().item() <= 5e-2 * ref.abs().max().item()
