"""BASELINE.json's five configurations (configs[0..4]) as workload records.

Configuration data only (kind, extents, T); the values are drawn by synth.make_inputs.
"""
from dataclasses import dataclass

from . import K7C, K7V, K25W, K25V, K25WA


@dataclass(frozen=True)
class Workload:
    name: str
    kind: int
    nx: int
    ny: int
    nz: int
    T: int

    @property
    def luops(self) -> int:
        """Lattice updates of one run: nx*ny*nz*T (interior only; reading Q12)."""
        return self.nx * self.ny * self.nz * self.T


C1 = Workload("C1-7pt-const-64", K7C, 64, 64, 64, 10)
C2 = Workload("C2-7pt-var-512", K7V, 512, 512, 512, 100)
C3 = Workload("C3-25pt-wave-512", K25W, 512, 512, 512, 100)
C4 = Workload("C4-25pt-var-512", K25V, 512, 512, 512, 100)
C5 = Workload("C5-25pt-var-1024", K25V, 1024, 1024, 1024, 200)

CONFIGS = [C1, C2, C3, C4, C5]
# SURVEY.md NEXT-1 (not a BASELINE.json config): C3's wave with the domain-sized alpha field of Fig. 1e.
C3A = Workload("C3A-25pt-wave-alpha-512", K25WA, 512, 512, 512, 100)
EXTRA = [C3A]
BY_NAME = {w.name: w for w in CONFIGS + EXTRA}


def weak_c5(n_gpus: int) -> Workload:
    """C5 weak-scaling variant: 1024 x 1024 x (256 * n_gpus), T = 200 (reading Q17)."""
    return Workload(f"C5w-25pt-var-1024x1024x{256 * n_gpus}", K25V, 1024, 1024, 256 * n_gpus, 200)
