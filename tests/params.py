"""Algorithm parameters used by the tests, written out once here and handed to
BOTH sides (the oracle's OracleConfig and the library's hjcd_config).  These
are the DESIGN.md "Readings" defaults; test_abi checks that
hjcd_config_default() returns the same values."""
import math

DEFAULTS = dict(
    M=1000, K=50, B=100, ccd_iters=64, lm_iters=128,
    eps_p_coarse=5e-3, eps_o_coarse=5e-2,          # R12
    eps_p_fine=1e-6, eps_o_fine=1e-5,              # R26
    gamma=1e-6, delta0=1.0, delta_rho=0.98, delta_min=0.1,   # R10, R5
    sigma_ccd=0.05, sigma_rep=0.02, sigma_lm=0.05,           # R11, R15, R25
    lambda_=1e-3, d_floor=1e-8, R=0.5, beta=2.0, A=8,         # R20-R22
    w_p=1.0, w_o=0.5,                                        # R17
    succ_p=1e-3, succ_o=math.pi / 180.0,
    tau_deg=1e-5,                                            # R4
    rng_seed=0, repl_noise_all=0,
    target_early_exit=1,                                     # R26b
    ccd_early_exit=1,                                        # R12b
)


def params(**over):
    p = dict(DEFAULTS)
    p.update(over)
    p["lambda"] = p.pop("lambda_")
    return p


# C1 (BASELINE.json configs[0]): Panda, 1 target, M=64, K=8, B=16, fixed iterations
C1 = dict(M=64, K=8, B=16, ccd_iters=64, lm_iters=32)
