"""Latent parity gates of the GPU tests.

The bf16 pipeline has a precision floor: the oracle with every matmul operand
and output rounded to bf16 (oracle.pab_oracle emulate_bf16) differs from the
fp32 oracle by (scripts/bf16_floor.py, worst step, relL2 / max|d|/max|ref|):

    config                     unguided              guided (CFG g=4)
    smoke  L2 D144 T8 S256     4.2e-3 / 4.7e-3       1.57e-2 / 1.84e-2
    dh72   L2 D288 T4 S128     -                     1.57e-2 / 1.75e-2
    C1     L4 D144 T8 S1024    4.6e-3 / 5.5e-3       -
    C2 slice L1 full width     -                     1.24e-2 / 1.77e-2
    C3 slice L1 full width     -                     1.22e-2 / 1.77e-2
    C4 slice L1 full width     -                     1.22e-2 / 1.79e-2

CFG amplifies the eps rounding (eps_u + 4 (eps_c - eps_u)), hence the guided
floor.  Guided runs are held to 1.5x the worst measured guided floor; unguided
runs to the SURVEY.md 8c gate (1.5e-2 / 2%, ~3x their floor).
"""
REL_TOL, MAX_TOL = 1.5e-2, 2e-2
REL_TOL_CFG, MAX_TOL_CFG = 2.4e-2, 2.8e-2
