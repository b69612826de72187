"""Precision tiers  (oracle; test infrastructure).

Table 1 of the paper gives, per requested precision eps,
the PSWF parameter c, the number of Fourier modes per dimension N_1 = 2 n_f + 1
for the difference kernels, and the Chebyshev order p.  We take c, N_1 and p
verbatim.  The Fourier spacing is our reading R2: h_l = 2 pi/(3 r_l),
i.e. period 3 r_l, which is what the colleague geometry of Eq. 3.39 needs; the
table's h_0 = 1.33 pi (= 4 pi/3, Eq. 3.30) is off by the factor 2 of a
half-width box convention.  With that spacing the table's N_1 and p reproduce
eps (tests/test_oracle_kernels.py pins this).

Root level (reading R4): windowed M_1, truncation radius R_T = (1 + sqrt d) r_0
(PAPER.md:2485), period P_0 = 1 + R_T + r_1, n_f0 = ceil(2 c P_0 / (2 pi)).
Precisions not in the table snap to the next tighter tabulated one.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

# (eps, c, N_1, p)  -- PAPER.md:2028-2031
TABLE1 = [
    (1e-3, 7.2462000846862793, 13, 9),
    (1e-6, 13.739999771118164, 25, 18),
    (1e-9, 20.736000061035156, 39, 28),
    (1e-12, 27.870000839233398, 53, 38),
]


@dataclass(frozen=True)
class Params:
    eps: float
    c: float
    nf: int          # difference-kernel Fourier half-width, N_1 = 2 nf + 1
    p: int           # Chebyshev order
    RT: float        # root window truncation radius
    P0: float        # root Fourier period
    nf0: int         # root Fourier half-width

    def h(self, l: int) -> float:
        """Fourier spacing at level l (l = 0: root window)."""
        if l == 0:
            return 2.0 * math.pi / self.P0
        return 2.0 * math.pi / (3.0 * 2.0 ** (-l))

    def nfl(self, l: int) -> int:
        return self.nf0 if l == 0 else self.nf


def for_eps(eps: float, d: int = 3) -> Params:
    row = None
    for r in TABLE1:                       # the loosest row at least as tight as eps
        if r[0] <= eps * (1 + 1e-9):
            row = r
            break
    if row is None:
        raise ValueError(f"eps={eps} tighter than Table 1 supports")
    e, c, N1, p = row
    RT = 1.0 + math.sqrt(d)            # (1 + sqrt d) r_0
    P0 = 1.0 + RT + 0.5
    nf0 = int(math.ceil(2.0 * c * P0 / (2.0 * math.pi)))
    return Params(eps=e, c=c, nf=(N1 - 1) // 2, p=p, RT=RT, P0=P0, nf0=nf0)
