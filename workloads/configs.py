"""The five BASELINE.json configurations as plain parameter records.

Overlap choices follow SURVEY.md §8(c) C-8 (recorded in DESIGN.md):
  c1 FixedNodes(1); c2 GL Relative(0.09)+floor 1 (Table 1 row 13);
  c3, c4 GLL Relative(0.08) (Table 1 row 3);
  c5 MaxRelative(0.08)+floor 1 (Table 2 "0.08 max").
Penalty (the ABI's `penalty` is the factor on the coercivity threshold P(P+1)/(2 Delta), reading
R2): factor 2 = the paper's "mu = 2 mu_min" with mu_min the stability threshold
for c2-c5; c1 states "penalty mu as defined in SPEC.md", i.e. 2 x the printed example
P(P+1)/Delta, which is factor 4 here.
"""
from dataclasses import dataclass, field
import math

GLL, GL = 0, 1
OVL_NODES, OVL_REL, OVL_MAXREL = 0, 1, 2


@dataclass(frozen=True)
class OverlapSpec:
    mode: int          # OVL_NODES / OVL_REL / OVL_MAXREL
    value: float       # n_o for OVL_NODES, alpha otherwise
    floor: int = 0     # minimum node layers


@dataclass(frozen=True)
class Config:
    name: str
    ne: tuple          # elements per direction (nx, ny, nz)
    length: tuple      # (lx, ly, lz)
    P: int
    basis: int
    overlap: OverlapSpec
    penalty: float = 2.0
    rhs: str = "uniform"        # "uniform" (seeded, zero mean) or "sin" (3 sin x sin y sin z)
    run: str = "vcycle"         # "vcycle" | "solve" | "pcg"
    cycles: int = 1
    rtol: float = 1e-10
    extra: dict = field(default_factory=dict)

    @property
    def nelem(self):
        return self.ne[0] * self.ne[1] * self.ne[2]

    @property
    def ndofs(self):
        return self.nelem * (self.P + 1) ** 3


TWO_PI = 2.0 * math.pi

CONFIGS = {
    "c1": Config("c1", (4, 4, 4), (1.0, 1.0, 1.0), 4, GLL, OverlapSpec(OVL_NODES, 1, 0),
                 penalty=4.0, run="vcycle", cycles=1),        # mu = 2 P(P+1)/Delta
    "c2": Config("c2", (8, 8, 8), (TWO_PI, TWO_PI, TWO_PI), 8, GL, OverlapSpec(OVL_REL, 0.09, 1),
                 rhs="sin", run="solve", cycles=30),
    "c3": Config("c3", (16, 16, 16), (1.0, 1.0, 1.0), 16, GLL, OverlapSpec(OVL_REL, 0.08, 0),
                 run="vcycle", cycles=5),
    "c4": Config("c4", (4, 4, 4), (1.0, 1.0, 1.0), 32, GLL, OverlapSpec(OVL_REL, 0.08, 0),
                 run="vcycle", cycles=5),
    "c5": Config("c5", (16, 16, 16), (48.0, 1.0, 1.0), 8, GL, OverlapSpec(OVL_MAXREL, 0.08, 1),
                 run="pcg", cycles=60),
}


def get_config(name, ne=None):
    """Return config `name`, optionally on a reduced element grid `ne` (same P/basis/overlap)."""
    c = CONFIGS[name]
    if ne is None:
        return c
    if isinstance(ne, int):
        ne = (ne, ne, ne)
    if c.rhs == "sin":
        length = c.length          # the sin-product RHS needs the 2*pi-periodic box
    else:
        # keep the element shape (and so the overlap resolution) identical
        length = tuple(c.length[d] * ne[d] / c.ne[d] for d in range(3))
    return Config(c.name + "-ne%dx%dx%d" % ne, tuple(ne), length, c.P, c.basis, c.overlap,
                  c.penalty, c.rhs, c.run, c.cycles, c.rtol, dict(c.extra))
