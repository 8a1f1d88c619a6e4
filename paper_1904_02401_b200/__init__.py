"""B200-native MG-GMRES / Vanka linear-solve path of the approximated-Newton
ALE-FSI solver (arXiv 1904.02401), drop-in for the reference's
``alefsi.linsolve`` / ``alefsi.newton.LinearStack`` solver entry points."""

__version__ = "0.1.0"
