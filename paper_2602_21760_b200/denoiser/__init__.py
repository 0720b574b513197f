"""Neural denoisers behind the seam (reference mixture.py:152-158 /
engine.py:164-184): random-init SDXL-shaped U-Net and SD3-shaped MMDiT built
on the package's own sm_100a kernels (tcgen05 GEMM / implicit-GEMM conv,
fused attention, group/layer norm)."""
