"""The hand-written leading-eigenpair solver of the POD (k_pod.cu: block
subspace iteration with CholQR and Rayleigh-Ritz / one-CTA Jacobi) against
LAPACK (numpy eigh, the oracle's dsyevd) and against cuSOLVER syevd
(PODECM_POD_EIG=syevd): the order-<=128 path (Jacobi on the Gram itself), the
subspace path, and a rank-deficient snapshot set (repeated snapshots: the
CholQR pivot guard).  Eigenvalues within 1e-10 relative, modes within 1e-8
up to sign, orthonormal after the MGS pass."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sign_fix(M):
    idx = np.abs(M).argmax(0)
    return M * np.sign(M[idx, np.arange(M.shape[1])])


def _snap(n_dof, L, rank, seed):
    rng = np.random.default_rng(seed)
    basis = rng.standard_normal((n_dof, rank)) * (1.0 / (1.0 + np.arange(rank)))  # decaying spectrum
    coef = rng.standard_normal((rank, L))
    return basis @ coef


@pytest.mark.parametrize("n_dof,L,rank,k", [(3000, 100, 100, 12), (5000, 600, 600, 50), (4000, 300, 150, 20)])
def test_pod_eig_against_lapack_and_syevd(monkeypatch, n_dof, L, rank, k):
    import torch
    from oracle import pod_ecm
    from paper_2307_16894_b200 import api
    S = _snap(n_dof, L, rank, n_dof + L)
    if rank < L:
        S[:, rank:] = S[:, : L - rank]  # repeated snapshots: Gram of rank `rank`
    St = torch.from_numpy(np.ascontiguousarray(S.T)).cuda()
    monkeypatch.delenv("PODECM_POD_EIG", raising=False)
    mg, eg = api.pod(St, k)
    monkeypatch.setenv("PODECM_POD_EIG", "syevd")
    ms, es = api.pod(St, k)
    mo, lo = pod_ecm.pod_diag(S, None, k)
    eg, es = eg.cpu().numpy()[:k], es.cpu().numpy()[:k]
    rel = np.abs(eg - lo[:k]) / lo[:k]
    rel_s = np.abs(eg - es) / es
    gm = _sign_fix(mg.cpu().numpy().T)
    dm = np.abs(gm - _sign_fix(mo)).max() / np.abs(mo).max()
    ds = np.abs(gm - _sign_fix(ms.cpu().numpy().T)).max() / np.abs(mo).max()
    print(f"n_snap {L} rank {rank} k {k}: eig vs LAPACK {rel.max():.2e}, vs syevd {rel_s.max():.2e}; "
          f"modes vs LAPACK {dm:.2e}, vs syevd {ds:.2e}")
    assert rel.max() <= 1e-10 and rel_s.max() <= 1e-10
    assert dm <= 1e-8 and ds <= 1e-8
    assert np.abs(gm.T @ gm - np.eye(k)).max() <= 1e-12
