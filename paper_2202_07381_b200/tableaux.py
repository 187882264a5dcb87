"""Butcher tableaux for the stage-coupled systems (host-side constants).

Only the s x s matrix ``A`` enters the hot path (the Kronecker factor of
the stage operator, stages.py:110-126).  Coefficients are evaluated with the
same closed forms as the reference registry (tableaux.py:48-111) so the
device sees bit-identical ``a_ij``.
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["ButcherTableau", "tableau_lookup", "registry_keys"]

_R3 = np.sqrt(3.0)
_R6 = np.sqrt(6.0)
_R15 = np.sqrt(15.0)


@dataclass(frozen=True)
class ButcherTableau:
    name: str
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray

    def __post_init__(self):
        for f in ("A", "b", "c"):
            object.__setattr__(self, f, np.asarray(getattr(self, f), dtype=np.float64))

    @property
    def r(self):
        return len(self.b)


def _gauss(s):
    if s == 1:
        return ButcherTableau("Gauss(1)", [[0.5]], [1.0], [0.5])
    if s == 2:
        return ButcherTableau("Gauss(2)",
                              [[1 / 4, 1 / 4 - _R3 / 6], [1 / 4 + _R3 / 6, 1 / 4]],
                              [1 / 2, 1 / 2], [1 / 2 - _R3 / 6, 1 / 2 + _R3 / 6])
    if s == 3:
        return ButcherTableau("Gauss(3)", [
            [5 / 36, 2 / 9 - _R15 / 15, 5 / 36 - _R15 / 30],
            [5 / 36 + _R15 / 24, 2 / 9, 5 / 36 - _R15 / 24],
            [5 / 36 + _R15 / 30, 2 / 9 + _R15 / 15, 5 / 36],
        ], [5 / 18, 4 / 9, 5 / 18], [1 / 2 - _R15 / 10, 1 / 2, 1 / 2 + _R15 / 10])
    raise KeyError


def _radau(s):
    if s == 1:
        return ButcherTableau("RadauIIA(1)", [[1.0]], [1.0], [1.0])
    if s == 2:
        return ButcherTableau("RadauIIA(2)", [[5 / 12, -1 / 12], [3 / 4, 1 / 4]],
                              [3 / 4, 1 / 4], [1 / 3, 1.0])
    if s == 3:
        return ButcherTableau("RadauIIA(3)", [
            [(88 - 7 * _R6) / 360, (296 - 169 * _R6) / 1800, (-2 + 3 * _R6) / 225],
            [(296 + 169 * _R6) / 1800, (88 + 7 * _R6) / 360, (-2 - 3 * _R6) / 225],
            [(16 - _R6) / 36, (16 + _R6) / 36, 1 / 9],
        ], [(16 - _R6) / 36, (16 + _R6) / 36, 1 / 9], [(4 - _R6) / 10, (4 + _R6) / 10, 1.0])
    raise KeyError


def _lobatto(s):
    if s == 2:
        return ButcherTableau("LobattoIIIC(2)", [[1 / 2, -1 / 2], [1 / 2, 1 / 2]],
                              [1 / 2, 1 / 2], [0.0, 1.0])
    if s == 3:
        return ButcherTableau("LobattoIIIC(3)",
                              [[1 / 6, -1 / 3, 1 / 6], [1 / 6, 5 / 12, -1 / 12],
                               [1 / 6, 2 / 3, 1 / 6]],
                              [1 / 6, 2 / 3, 1 / 6], [0.0, 1 / 2, 1.0])
    raise KeyError


def _backward_euler(s):
    if s != 1:
        raise KeyError
    return ButcherTableau("BackwardEuler", [[1.0]], [1.0], [1.0])


def _dirk2(s):
    if s != 2:
        raise KeyError
    g = 1.0 - np.sqrt(2.0) / 2.0
    return ButcherTableau("DIRK-PareschiRusso(2)", [[g, 0.0], [1.0 - 2.0 * g, g]],
                          [1 / 2, 1 / 2], [g, 1.0 - g])


def _dirk3(s):
    """Alexander's 3-stage L-stable SDIRK (tableaux.py:98-111): the diagonal
    g is the root of g^3 - 3 g^2 + 3/2 g - 1/6 in (1/6, 1/2), taken from the
    companion-matrix roots as the reference does (same bits)."""
    if s != 3:
        raise KeyError
    cand = [z.real for z in np.roots([1.0, -3.0, 1.5, -1.0 / 6.0])
            if abs(z.imag) < 1e-12 and 0.0 < z.real < 0.5]
    g = float(min(cand))
    tau = 0.5 * (1.0 + g)
    b1 = -(6.0 * g * g - 16.0 * g + 1.0) / 4.0
    b2 = (6.0 * g * g - 20.0 * g + 5.0) / 4.0
    return ButcherTableau("DIRK-Alexander(3)", [[g, 0.0, 0.0], [tau - g, g, 0.0], [b1, b2, g]],
                          [b1, b2, g], [g, tau, 1.0])


_FAMILIES = {"gauss": _gauss, "radauiia": _radau, "lobattoiiic": _lobatto,
             "backwardeuler": _backward_euler, "dirk-pareschirusso": _dirk2,
             "dirk-alexander": _dirk3}
_ALIASES = {"radau": "radauiia", "lobatto": "lobattoiiic", "be": "backwardeuler",
            "dirk2": "dirk-pareschirusso", "pareschirusso": "dirk-pareschirusso",
            "alexander": "dirk-alexander", "dirk3": "dirk-alexander"}


def tableau_lookup(family, stages):
    """Tableau for (family, stages); KeyError if unsupported (tableaux.py:137-146)."""
    key = family.strip().lower().replace("_", "-")
    key = _ALIASES.get(key, key)
    if key not in _FAMILIES:
        raise KeyError(f"unknown tableau family {family!r}")
    try:
        return _FAMILIES[key](int(stages))
    except KeyError:
        raise KeyError(f"family {family!r} does not provide a {stages}-stage scheme") from None


def registry_keys():
    return [("gauss", 1), ("gauss", 2), ("gauss", 3), ("radauiia", 1), ("radauiia", 2),
            ("radauiia", 3), ("lobattoiiic", 2), ("lobattoiiic", 3), ("backwardeuler", 1),
            ("dirk-pareschirusso", 2), ("dirk-alexander", 3)]
