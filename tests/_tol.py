"""The numerics bars every test enforces, with the bound each one comes from
(DESIGN.md section 2 states the same numbers).

* fp32 AG path: bitwise against reference::gemm (reference.hpp:36-49).
* placement (gathered operand, FD wire rows' locations): bit-exact.
* FD_F32_REF: the reference's own head-relative bar for its fp32 path
  (flash_decode_test.cpp:63-88) -- our fp32 (generic-kernel) path meets it.
* FD_F32: bf16 K/V decoded on tensor cores with fp32 output.  The weights P
  reach the PV product as a bf16 hi + lo pair (P = hi + lo to ~2^-16) and
  everything else accumulates in fp32: measured 3.5e-6 (config 3) and
  1.1e-5 (config 4) against fp32 torch; bar 1e-4.
* FD_BF16: the same path with bf16 output.  A bf16 element's own
  round-to-nearest error is at most half an ulp, 2^-8 of the element's
  binade, i.e. <= 2^-8 (3.906e-3) of the head's max |o| -- so the bar is
  2^-8 plus the fp32-grade path's FD_F32.  Measured 3.5e-3 - 3.9e-3.
* AG_BF16: bf16 C of an fp32-accumulated tcgen05 GEMM: the same 2^-8
  output rounding of max|C| plus fp32 accumulation error (~1e-6): 4e-3.
"""
FD_F32_REF = 1e-5
FD_F32 = 1e-4
FD_BF16 = 2.0 ** -8 + FD_F32
AG_BF16 = 4e-3
