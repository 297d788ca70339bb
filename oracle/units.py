"""Physical constants of the oracle (units nm, ps, u, kJ/mol, e, K)."""
import math

F_COUL = 138.935458          # 1/(4 pi eps0) in kJ mol^-1 nm e^-2
KB = 0.0083144626            # kJ mol^-1 K^-1
LN10 = math.log(10.0)


def kT(T):
    return KB * T
