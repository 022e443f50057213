"""Comparison metrics for the parity tests (readings R8, R9).

* floored elementwise relative error:
      e = max_{i>=j} |Lg_ij - Lo_ij| / max(|Lo_ij|, 1e-4 * sqrt(A_ii))
  The literal "max elementwise relative error" of north_star is ill-posed for
  entries that are ~1e-8 of their row scale; since ||L_i,:||_2 = sqrt(A_ii),
  the floor is 1e-4 of the largest possible entry of row i.
* backward error (north_star): ||A - L L^T||_F / (n * eps * ||A||_F), eps = 2^-52.
"""
import numpy as np

EPS = 2.0 ** -52


def lower_of(F: np.ndarray, uplo: str) -> np.ndarray:
    """The factor in L-view (n x n lower) from a column-major result matrix."""
    F = np.asarray(F)
    return np.tril(F) if uplo.upper() == "L" else np.tril(F.T)


def floored_rel_err(Lg: np.ndarray, Lo: np.ndarray, A: np.ndarray) -> float:
    Lg = np.tril(Lg)
    Lo = np.tril(Lo)
    n = Lo.shape[0]
    if n == 0:
        return 0.0
    floor = 1e-4 * np.sqrt(np.abs(np.diag(A)))[:, None]
    den = np.maximum(np.abs(Lo), floor)
    return float(np.max(np.tril(np.abs(Lg - Lo) / den)))


def backward_error(A_sym: np.ndarray, L: np.ndarray) -> float:
    n = A_sym.shape[0]
    if n == 0:
        return 0.0
    L = np.tril(L)
    R = A_sym - L @ L.T
    return float(np.linalg.norm(R) / (n * EPS * np.linalg.norm(A_sym)))


def sym_from(A: np.ndarray, uplo: str) -> np.ndarray:
    """Full symmetric matrix rebuilt from the uplo triangle only."""
    T = np.tril(A) if uplo.upper() == "L" else np.triu(A)
    D = np.diag(np.diag(T))
    return T + T.T - D
