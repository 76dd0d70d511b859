"""Plain CPU CP-ALS / MSDT / pairwise-perturbation oracle (NumPy/SciPy, float64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): never imported by the
product package.  Citations: ``P:n`` = /root/reference/PAPER.md line n.

Layout convention (reading R2): tensors are
row-major (last mode fastest).  ``unfold(T, n)`` keeps mode n as rows and the
remaining modes in ascending order, last fastest; the matching Khatri-Rao
product takes the factors in ascending mode order with the FIRST operand's row
index slowest.  This is the same product T_(n) P^(n) as the paper's Kolda
ordering "A^(N) ⊙ ... ⊙ A^(1)" with the first mode fastest;
the elementwise definition (brute force in the pins) is convention-free.
"""
from __future__ import annotations

import dataclasses
import itertools
import math

import numpy as np
import scipy.linalg as sla

import synth

__all__ = [
    "unfold", "khatri_rao", "mttkrp", "gram", "gamma", "solve", "norm2", "fitness_eq3",
    "residual_eq2", "kruskal", "make_tensor", "make_tensor_block", "make_tensor_slice", "mttkrp_rows",
    "als_sweep", "PPState", "pp_init", "pp_approx_sweep", "pp_condition", "pp_controller_run",
    "ttm", "block_contract", "mttv", "MSDTModel", "DTModel", "msdt_roots", "par_als_sweep_sim",
    "par_pp_approx_sweep_sim", "dS_of", "pp_first_order", "pp_second_order", "eq3_radicand",
    "RADICAND_TOL", "pp_init_rows", "pp_approx_rows", "grid_procs", "par_als_sweep_grid_sim",
    "par_pp_approx_sweep_grid_sim",
]


# ---------------------------------------------------------------------------
# Notation and definitions (§II-A; §II-B)
# ---------------------------------------------------------------------------

def unfold(T, n):
    """Mode-n matricization T_(n): rows = mode n, columns = the other
    modes in ascending order with the last one fastest (row-major)."""
    return np.ascontiguousarray(np.moveaxis(T, n, 0)).reshape(T.shape[n], -1)


def khatri_rao(mats):
    """Khatri-Rao product: column k is the Kronecker product of the
    k-th columns; (a ⊗ b)(i*J + j) = a(i) b(j) -- first operand slowest."""
    R = mats[0].shape[1]
    out = mats[0]
    for B in mats[1:]:
        out = (out[:, None, :] * B[None, :, :]).reshape(-1, R)
    return out


def mttkrp(T, A, n, block_rows=None):
    """MTTKRP M^(n) = T_(n) P^(n) with an explicitly formed Khatri-Rao product
    P^(n).  `block_rows` forms P^(n) in row blocks of the
    unfolding's column space to bound memory (still explicit)."""
    N = T.ndim
    others = [A[m] for m in range(N) if m != n]
    Tn = unfold(T, n)
    if block_rows is None or len(others) < 2:
        return Tn @ khatri_rao(others)
    # explicit KRP in blocks of its leading factor's rows
    lead, rest = others[0], khatri_rao(others[1:])
    K = rest.shape[0]
    M = np.zeros((T.shape[n], A[0].shape[1]))
    for i0 in range(0, lead.shape[0], block_rows):
        blk = khatri_rao([lead[i0:i0 + block_rows], rest])
        M += Tn[:, i0 * K:(i0 + blk.shape[0] // K) * K] @ blk
    return M


def gram(A):
    """S = A^T A.  Upper triangle computed, then mirrored, so S is exactly symmetric."""
    S = A.T @ A
    iu = np.triu_indices(S.shape[0], 1)
    S[(iu[1], iu[0])] = S[iu]
    return S


def gamma(S, n):
    """Γ^(n) = S^(1) * ... * S^(n-1) * S^(n+1) * ... * S^(N) (Eq. 1)."""
    G = np.ones_like(S[0])
    for k, Sk in enumerate(S):
        if k != n:
            G = G * Sk
    return G


def solve(G, M):
    """A^(n) <- M^(n) Γ^(n)† (Alg. 1 line 7) as a Cholesky solve (reading Q3:
    Γ is SPD for full-column-rank factors)."""
    c = sla.cho_factor(G, lower=True)
    return np.ascontiguousarray(sla.cho_solve(c, M.T).T)


def norm2(T):
    """||T||_F^2, computed once."""
    return float(np.dot(T.ravel(), T.ravel()))


def eq3_radicand(normT2, G_N, S_N, M_N, A_N):
    """The quantity under the root of Eq. 3, ||T||^2 + <Γ^(N), S^(N)> - 2<M^(N), A^(N)>
    (reading Q1: ||T||^2, the printed unsquared norm is a typo).  It equals ||T - T~||^2 when M^(N)
    is the exact MTTKRP; with an approximated M~^(N) it can be negative (reading R18)."""
    return normT2 + float(np.sum(G_N * S_N)) - 2.0 * float(np.sum(M_N * A_N))


def fitness_eq3(normT2, G_N, S_N, M_N, A_N):
    """Relative residual from Eq. 3 and f = 1 - r; a negative radicand is
    clamped to 0.  Returns (f, r)."""
    rad = eq3_radicand(normT2, G_N, S_N, M_N, A_N)
    r = math.sqrt(max(rad, 0.0)) / math.sqrt(normT2)
    return 1.0 - r, r


RADICAND_TOL = 1e-8   # Eq. 3 radicand below -RADICAND_TOL ||T||^2: not a residual (reading R18)


def kruskal(A):
    """[[A^(1), ..., A^(N)]] = Σ_r A^(1)(:,r) ∘ ... ∘ A^(N)(:,r)."""
    R = A[0].shape[1]
    out = None
    for r in range(R):
        t = A[0][:, r]
        for B in A[1:]:
            t = np.multiply.outer(t, B[:, r])
        out = t if out is None else out + t
    return out


def residual_eq2(T, A):
    """r = ||T - T~||_F / ||T||_F with an explicit reconstruction (Eq. 2)."""
    D = T - kruskal(A)
    return math.sqrt(norm2(D) / norm2(T))


# ---------------------------------------------------------------------------
# Synthetic tensors (independent reconstruction; the hash comes from synth)
# ---------------------------------------------------------------------------

def _index_grid(shape, ranges):
    """Global linear indices (uint64) of the sub-block `ranges` of a tensor of `shape`."""
    idx = np.zeros([hi - lo for lo, hi in ranges], dtype=np.uint64)
    stride = 1
    for d in reversed(range(len(shape))):
        lo, hi = ranges[d]
        ax = np.arange(lo, hi, dtype=np.uint64) * np.uint64(stride)
        sh = [1] * len(shape)
        sh[d] = hi - lo
        idx = idx + ax.reshape(sh)
        stride *= shape[d]
    return idx


def make_tensor_block(cfg, ranges):
    """T restricted to the index box `ranges` (list of [lo,hi) per mode):
    Kruskal part of the true factors plus the seeded noise, or the
    seeded U(0,1) entries for the structureless config (synth recipe)."""
    idx = _index_grid(cfg.shape, ranges)
    noise = synth.element_noise(cfg, idx)
    if cfg.kind == "uniform":
        return noise
    At = synth.true_factors(cfg)
    return kruskal([a[lo:hi] for a, (lo, hi) in zip(At, ranges)]) + noise


def make_tensor(cfg, rank=0, world=1):
    """Local slab of T for `rank` of a 1-D partition along the last mode."""
    shape = cfg.shape
    lo, hi = synth.slab_range(shape[-1], rank, world)
    ranges = [(0, d) for d in shape[:-1]] + [(lo, hi)]
    return make_tensor_block(cfg, ranges)


def make_tensor_slice(cfg, n, i):
    """The (N-1)-way slice T(..., i_n = i, ...) (for row-sampled MTTKRP checks)."""
    shape = cfg.shape
    ranges = [(0, d) for d in shape]
    ranges[n] = (i, i + 1)
    return make_tensor_block(cfg, ranges).reshape([d for m, d in enumerate(shape) if m != n])


def mttkrp_rows(cfg, A, n, rows):
    """Rows `rows` of M^(n) computed slice by slice with the explicit KRP:
    M^(n)(i,:) = vec(T(...,i,...))^T P^(n)."""
    others = [A[m] for m in range(cfg.N) if m != n]
    lead, rest = others[0], khatri_rao(others[1:])   # explicit KRP, formed per lead row
    K = rest.shape[0]
    out = []
    for i in rows:
        sl = make_tensor_slice(cfg, n, int(i)).reshape(lead.shape[0], K)
        out.append(sum(sl[a] @ khatri_rao([lead[a:a + 1], rest]) for a in range(lead.shape[0])))
    return np.stack(out)


# ---------------------------------------------------------------------------
# Exact CP-ALS sweep (Alg. 1) -- this IS msdt_sweep and dt_sweep
# (MSDT/DT are exact reorganisations)
# ---------------------------------------------------------------------------

def als_sweep(T, A, normT2=None):
    """One CP-ALS sweep (Alg. 1 lines 5-9) with direct MTTKRPs, then Eq. 3.

    Returns dict(A=new factors, S=Grams, M=[M^(n)], dA=[per-sweep update],
    G=[Γ^(n)], f=fitness, r=residual).
    """
    N = T.ndim
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    if normT2 is None:
        normT2 = norm2(T)
    Ms, dA, Gs = [], [], []
    for n in range(N):
        G = gamma(S, n)
        M = mttkrp(T, A, n)
        new = solve(G, M)
        dA.append(new - A[n])
        A[n] = new
        S[n] = gram(new)
        Ms.append(M)
        Gs.append(G)
    f, r = fitness_eq3(normT2, Gs[-1], S[-1], Ms[-1], A[-1])
    rad = eq3_radicand(normT2, Gs[-1], S[-1], Ms[-1], A[-1]) / normT2
    return dict(A=A, S=S, M=Ms, dA=dA, G=Gs, f=f, r=r, rad=rad)


# ---------------------------------------------------------------------------
# Pairwise perturbation (§II-C, Eqs. 4-8, Alg. 2)
# ---------------------------------------------------------------------------

@dataclasses.dataclass
class PPState:
    Ap: list                 # A_p^(i) snapshot (Alg. 2 line 7)
    ops: dict                # (a,b) a<b -> M_p^(a,b) as [s_a, s_b, R]  (Eq. 4 with A_p)
    Mp: list                 # M_p^(n) = exact MTTKRP at A_p


def pp_init(T, A):
    """PP initialisation (Alg. 2 lines 6-9): A_p <- A, dA <- 0, and the
    operators M_p^(a,b) = T_(a,b) ⊙_{m∉{a,b}} A_p^(m) (Eq. 4), computed
    directly with explicit partial Khatri-Rao products (not via the PP tree)."""
    N = T.ndim
    Ap = [a.copy() for a in A]
    ops = {}
    for a, b in itertools.combinations(range(N), 2):
        rest = [m for m in range(N) if m not in (a, b)]
        Tab = np.ascontiguousarray(np.moveaxis(T, (a, b), (0, 1))).reshape(T.shape[a], T.shape[b], -1)
        ops[(a, b)] = Tab @ khatri_rao([Ap[m] for m in rest])
    Mp = [mttkrp(T, Ap, n) for n in range(N)]
    return PPState(Ap=Ap, ops=ops, Mp=Mp)


def pp_init_rows(cfg, Ap, n, rows, slices=None):
    """The part of PP initialisation (Alg. 2 lines 6-9; Eq. 4) that Eq. 5 needs for the
    rows `rows` of mode n: M_p^(n,i)(x, y, k) for x in rows and every i != n, and M_p^(n)(x, :),
    each from the slice T(..., i_n = x, ...) with an explicit partial Khatri-Rao product of the
    other A_p^(m) (for full-size tensors whose pair operators the oracle cannot hold).
    Returns a PPState whose operators are restricted to those rows (the pair {n, i} keeps its
    [s_a, s_b, R] orientation with mode n's axis cut to len(rows)), so pp_first_order applies
    unchanged.  `slices` (optional dict) caches T's slices across calls."""
    N, R = cfg.N, Ap[0].shape[1]
    ops, mp = {}, []
    for i in range(N):
        if i == n:
            continue
        rest = [m for m in range(N) if m not in (n, i)]
        krp = khatri_rao([Ap[m] for m in rest])
        blk = []
        for x in rows:
            key = (n, int(x))
            sl = slices.get(key) if slices is not None else None
            if sl is None:
                sl = make_tensor_slice(cfg, n, int(x))      # modes != n, ascending
                if slices is not None:
                    slices[key] = sl
            kept = [m for m in range(N) if m != n]
            Ti = np.ascontiguousarray(np.moveaxis(sl, kept.index(i), 0)).reshape(cfg.shape[i], -1)
            blk.append(Ti @ krp)                             # [s_i, R]
        blk = np.stack(blk)                                  # [rows, s_i, R]
        ops[(n, i) if n < i else (i, n)] = blk if n < i else np.ascontiguousarray(blk.transpose(1, 0, 2))
    # M_p^(n) rows: one more contraction of any pair operator row with A_p^(i) (Eq. 4 -> MTTKRP)
    i0 = 0 if n != 0 else 1
    op = ops[(n, i0) if n < i0 else (i0, n)]
    mp = np.einsum("xyk,yk->xk", op, Ap[i0]) if n < i0 else np.einsum("yxk,yk->xk", op, Ap[i0])
    Mp = [None] * N
    Mp[n] = mp
    return PPState(Ap=[a.copy() for a in Ap], ops=ops, Mp=Mp)


def pp_approx_rows(st_rows: PPState, A, n, rows):
    """M~^(n)(rows, :) of Eq. 5 at the current factors A (modes < n already updated
    this sweep): the first-order terms from the row-restricted operators, plus V^(n)(rows) =
    A^(n)(rows) W^(n) (Eqs. 7-8) with W^(n) from the full current factors."""
    N = len(A)
    dA = [A[i] - st_rows.Ap[i] for i in range(N)]
    S = [gram(a) for a in A]
    return pp_first_order(st_rows, dA, n) + A[n][rows] @ pp_second_order(A, dA, S, n)


def dS_of(A_i, dA_i):
    """dS^(i) = A^(i)T dA^(i) (Eq. 8); row index = model rank, not symmetrised."""
    return A_i.T @ dA_i


def pp_condition(dA, A, eps):
    """Alg. 2 line 5 / line 10: ∀i ||dA^(i)||_F < ε ||A^(i)||_F (strict)."""
    return all(np.linalg.norm(d) < eps * np.linalg.norm(a) for d, a in zip(dA, A))


def pp_first_order(st: PPState, dA, n):
    """M_p^(n) + Σ_{i≠n} U^(n,i) (Eqs. 5-6): U^(n,i)(x,k) = Σ_y M_p^(n,i)(x,y,k) dA^(i)(y,k);
    the pair {a<b} is stored once as [s_a, s_b, R] and contracted on the axis of mode i."""
    Mt = st.Mp[n].copy()
    for i in range(len(dA)):
        if i == n:
            continue
        if n < i:   # operator stored as [s_n, s_i, R]: contract its second axis
            Mt += np.einsum("xyk,yk->xk", st.ops[(n, i)], dA[i])
        else:       # stored as [s_i, s_n, R]: contract its first axis
            Mt += np.einsum("yxk,yk->xk", st.ops[(i, n)], dA[i])
    return Mt


def pp_second_order(A, dA, S, n):
    """W^(n) = Σ_{i<j; i,j≠n} dS^(i) * dS^(j) * ∗_{k∉{i,j,n}} S^(k) (Eq. 7; reading Q7:
    i, j range over {1..N}\\{n}) with dS^(i) = A^(i)T dA^(i) (Eq. 8).  The second-order
    term of Eq. 5 is V^(n) = A^(n) W^(n) (pre-update A^(n), reading Q8)."""
    N = len(A)
    dS = [dS_of(A[i], dA[i]) for i in range(N)]
    W = np.zeros_like(S[0])
    for i, j in itertools.combinations([m for m in range(N) if m != n], 2):
        term = dS[i] * dS[j]
        for k in range(N):
            if k not in (i, j, n):
                term = term * S[k]
        W += term
    return W


def pp_approx_sweep(st: PPState, A, normT2, eps=None):
    """One PP approximated sweep (Alg. 2 lines 11-16; Eqs. 5-8).

    For n = 1..N: Γ^(n); dA^(i) = A^(i) - A_p^(i) (current); U^(n,i) (Eq. 6);
    dS^(i) (Eq. 8); V^(n) = A^(n) W^(n) with W^(n) = Σ_{i<j; i,j≠n}
    dS^(i)*dS^(j)*∗_{k∉{i,j,n}} S^(k) (Eq. 7, reading Q7/Q8: all current, A^(n)
    pre-update); M~^(n) = M_p^(n) + Σ_i U^(n,i) + V^(n) (Eq. 5); solve; update
    dA^(n), S^(n).  Fitness by Eq. 3 with M~^(N) (reading Q21); `rad` is Eq. 3's
    radicand / ||T||^2 (negative: the sweep left M~ and A inconsistent, reading R18).
    Returns dict(A, S, M=[M~^(n)], V, f, r, rad, still_valid, dA).
    """
    N = len(A)
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    Ms, Vs, Gs = [], [], []
    for n in range(N):
        G = gamma(S, n)
        dA = [A[i] - st.Ap[i] for i in range(N)]
        Mt = pp_first_order(st, dA, n)
        V = A[n] @ pp_second_order(A, dA, S, n)
        Mt += V
        new = solve(G, Mt)
        A[n] = new
        S[n] = gram(new)
        Ms.append(Mt)
        Vs.append(V)
        Gs.append(G)
    f, r = fitness_eq3(normT2, Gs[-1], S[-1], Ms[-1], A[-1])
    rad = eq3_radicand(normT2, Gs[-1], S[-1], Ms[-1], A[-1]) / normT2
    dA = [A[i] - st.Ap[i] for i in range(N)]
    valid = pp_condition(dA, A, eps) if eps is not None else None
    return dict(A=A, S=S, M=Ms, V=Vs, f=f, r=r, rad=rad, still_valid=valid, dA=dA)


def pp_controller_run(T, A0, eps, delta=1e-5, max_sweeps=300, max_pp_run=None, stop_test="any"):
    """Alg. 2 driver; fitness after every sweep (reading Q21).

    Stop test: "any" (default, reading Q21) -- Δ between neighbouring sweeps of any kind (the
    P:931 wording); "regular" -- Alg. 2 as printed (lines 3-4, 19-21): r is
    updated only after a regular sweep and the loop ends when |r - r_old| <= Δ between consecutive
    regular sweeps (r = 1, r_old = 0 initially); approximated sweeps are traced, not tested.
    max_sweeps counts regular and approximated sweeps, not PP initialisations: the paper's
    iteration cap of 300 against Table 3's separate Num-ALS / Num-PP-init /
    Num-PP-approx columns.
    An approximated sweep whose Eq. 3 radicand is below -RADICAND_TOL ||T||^2 (reading R18) has no
    residual: its row carries fitness None, the PP run ends there (as if the ε test failed), and the
    Δ test skips it (the next regular sweep is compared with the last valid fitness).
    Returns (A, [(kind, f)])."""
    normT2 = norm2(T)
    A = [a.copy() for a in A0]
    dA = [a.copy() for a in A]          # Alg. 2 line 2: dA <- A
    trace, f_old = [], None
    f_reg_old = 0.0                     # r = 1 before the first regular sweep (line 3)
    n_sweeps = 0
    while n_sweeps < max_sweeps:
        stop = False
        if pp_condition(dA, A, eps):
            st = pp_init(T, A)
            trace.append(("pp_init", None))
            n_run = 0
            while True:
                out = pp_approx_sweep(st, A, normT2, eps)
                A = out["A"]
                n_sweeps += 1
                n_run += 1
                flagged = out["rad"] < -RADICAND_TOL
                trace.append(("pp_approx", None if flagged else out["f"]))
                if flagged:
                    break
                if stop_test == "any":
                    stop = f_old is not None and abs(out["f"] - f_old) <= delta
                f_old = out["f"]
                if stop or not out["still_valid"] or n_sweeps >= max_sweeps or \
                        (max_pp_run is not None and n_run >= max_pp_run):
                    break
            if stop or n_sweeps >= max_sweeps:
                break
        out = als_sweep(T, A, normT2)
        A, dA = out["A"], out["dA"]
        n_sweeps += 1
        trace.append(("regular", out["f"]))
        if stop_test == "any":
            if f_old is not None and abs(out["f"] - f_old) <= delta:
                break
        elif abs(out["f"] - f_reg_old) <= delta:
            break
        f_old = out["f"]
        f_reg_old = out["f"]
    return A, trace


# ---------------------------------------------------------------------------
# Dimension-tree schedule models (CPU models of the *schedules*, P:210-322 and
# §III).  They compute MTTKRPs through the trees with TTM/mTTV steps
# and are pinned against the direct MTTKRP under arbitrary factor updates.
# ---------------------------------------------------------------------------

def ttm(T, A, j):
    """First-level contraction T ×_j A^(j)T, output modes = the others (ascending) + R
    (Eq. 4 with one contracted mode)."""
    out = np.tensordot(T, A, axes=([j], [0]))        # moves the contracted axis out, R last
    return out


def block_contract(T, A, C):
    """Upper-level fusion ("combining several upper level contractions"): T contracted
    over all modes in C in ONE step, as the generalized unfolding T_(kept, C) (kept modes ascending,
    then C ascending, last fastest) times the explicit Khatri-Rao product of the factors of C in
    ascending mode order (first operand slowest, the convention of ``unfold``/``khatri_rao``).
    Output modes = the kept ones (ascending) + R."""
    C = sorted(C)
    kept = [m for m in range(T.ndim) if m not in C]
    Tm = np.ascontiguousarray(np.transpose(T, kept + C)).reshape(
        int(np.prod([T.shape[m] for m in kept], dtype=np.int64)), -1)
    K = khatri_rao([A[c] for c in C])
    return (Tm @ K).reshape([T.shape[m] for m in kept] + [K.shape[1]])


def mttv(X, v, axis):
    """Batched TTV: out[..., r] = Σ_y X[..., y, ..., r] v[y, r]."""
    Xm = np.moveaxis(X, axis, -2)                    # [..., y, r]
    return np.einsum("...yr,yr->...r", Xm, v)


def _split_contract(node, kept, drop_modes, A, order):
    """Contract the modes `drop_modes` of `node` (kept = its ascending mode list), one
    mTTV per mode, in `order` (service order, reading Q5)."""
    kept = list(kept)
    for m in order:
        if m in drop_modes:
            ax = kept.index(m)
            node = mttv(node, A[m], ax)
            kept.pop(ax)
    return node, kept


class _SubtreeRunner:
    """Lazy binary subtree (O3): served list L; left = first ceil(|L|/2) modes built by
    contracting the right modes (current), right = rest built by contracting the left
    modes after their updates.  Nodes are built just before first use."""

    def __init__(self, root, kept, served):
        self.served = list(served)
        self.cache = {(0, len(served)): (root, list(kept))}

    def leaf(self, q, A):
        L = self.served
        lo, hi = 0, len(L)
        node, kept = self.cache[(lo, hi)]
        while hi - lo > 1:
            mid = lo + (hi - lo + 1) // 2
            if q < mid:
                child, drop = (lo, mid), L[mid:hi]
            else:
                child, drop = (mid, hi), L[lo:mid]
            if child not in self.cache:
                self.cache[child] = _split_contract(node, kept, set(drop), A, L[lo:hi])
            lo, hi = child
            node, kept = self.cache[child]
        return node, kept


class MSDTModel:
    """MSDT schedule (§III, Fig. 2).  Root k (k = 0,1,...) is T ×_j A^(j) with
    j = N, N-1, ..., 1 cyclically (1-based; "root of ith subtree is T×_{N-i+1}"),
    serving the N-1 modes (j+1, ..., j+N-1) mod N (0≡N, reading Q4).  In a continuous
    stream of updates t = 0,1,..., mode(t) = t mod N and root k serves t in
    [k(N-1), (k+1)(N-1)).  Counts first-level TTMs (pin: N per N-1 sweeps).

    ``levels`` = l (upper-level fusion, P:700-702, 1 <= l <= N-2): root k contracts the l modes
    that follow its served block cyclically in ONE step (``block_contract``) and serves the
    N-l updates [k(N-l), (k+1)(N-l)), modes f, .., f+N-l-1 (mod N) with f = k(N-l) mod N;
    l = 1 is the schedule above (f + N-1 = j).  N roots per N-l sweeps."""

    def __init__(self, T, levels=1):
        self.T = T
        self.N = T.ndim
        if not 1 <= levels <= max(1, self.N - 2):
            raise ValueError("levels must be in [1, N-2]")
        self.l = levels
        self.t = 0
        self.runner = None
        self.n_ttm = 0
        self.trace = []      # (root contracted mode j (0-based) or the block C, served list)

    def next_mttkrp(self, A):
        N, l = self.N, self.l
        k, q = divmod(self.t, N - l)
        if q == 0:
            f = (k * (N - l)) % N
            served = [(f + d) % N for d in range(N - l)]
            C = [(f + d) % N for d in range(N - l, N)]
            if l == 1:
                j = C[0]                                  # = ((k + 1)(N - 1)) mod N
                root = ttm(self.T, A[j], j)
                self.trace.append((j, served))
            else:
                root = block_contract(self.T, A, C)
                self.trace.append((tuple(C), served))
            self.n_ttm += 1
            kept = [m for m in range(N) if m not in C]
            self.runner = _SubtreeRunner(root, kept, served)
        n = self.t % N
        node, kept = self.runner.leaf(q, A)
        assert kept == [n] and self.runner.served[q] == n
        self.t += 1
        return node


class DTModel:
    """Standard dimension tree (Fig. 1a; O4): per sweep, root T×_N then the
    modes ceil(N/2)+1..N-1 (current) serve 1..ceil(N/2); root T×_1 then modes
    2..ceil(N/2) (already updated) serve ceil(N/2)+1..N.  2 TTMs per sweep."""

    def __init__(self, T):
        self.T = T
        self.N = T.ndim
        self.n_ttm = 0
        self.n = 0
        self.runner = None

    def next_mttkrp(self, A):
        N = self.N
        h = (N + 1) // 2
        n = self.n % N
        if n == 0 or n == h:
            if n == 0:
                j, pre, served = N - 1, list(range(h, N - 1)), list(range(0, h))
            else:
                j, pre, served = 0, list(range(1, h)), list(range(h, N))
            node = ttm(self.T, A[j], j)
            self.n_ttm += 1
            kept = [m for m in range(N) if m != j]
            node, kept = _split_contract(node, kept, set(pre), A, pre)
            self.runner = _SubtreeRunner(node, kept, served)
            self.base = n
        q = n - self.base
        node, kept = self.runner.leaf(q, A)
        assert kept == [n]
        self.n += 1
        return node


def msdt_roots(N, n_sweeps):
    """Contracted mode (0-based) of every MSDT root used in `n_sweeps` sweeps."""
    n_updates = N * n_sweeps
    return [((k + 1) * (N - 1)) % N for k in range(-(-n_updates // (N - 1)))]


# ---------------------------------------------------------------------------
# Parallel algorithms on a 1-D grid 1x...x1xP (Alg. 3; Alg. 4)
# simulated in one process; the gloo test runs the same steps with real collectives.
# ---------------------------------------------------------------------------

def par_als_sweep_sim(T, A, P, normT2=None):
    """Alg. 3 with the tensor split along the last mode into P slabs: local MTTKRP
    (line 13) -> Reduce-Scatter (line 14, n<N) -> solve own rows (line 15) ->
    All-Gather A (line 18); mode N rows are local, S^(N) by All-Reduce (line 17)."""
    N = T.ndim
    sN = T.shape[-1]
    slabs = [T[..., lo:hi] for lo, hi in (synth.slab_range(sN, p, P) for p in range(P))]
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    if normT2 is None:
        normT2 = sum(norm2(t) for t in slabs)
    for n in range(N):
        G = gamma(S, n)
        loc = []
        for p, Tp in enumerate(slabs):
            lo, hi = synth.slab_range(sN, p, P)
            Ap = A[:-1] + [A[-1][lo:hi]]
            loc.append(mttkrp(Tp, Ap, n))
        if n < N - 1:
            M = sum(loc)                                   # reduce-scatter then all-gather
            b = T.shape[n] // P
            A[n] = np.concatenate([solve(G, M[p * b:(p + 1) * b]) for p in range(P)])
            S[n] = gram(A[n])
        else:
            M = np.concatenate(loc)
            A[n] = np.concatenate([solve(G, m) for m in loc])
            S[n] = sum(gram(A[n][synth.slab_range(sN, p, P)[0]:synth.slab_range(sN, p, P)[1]])
                       for p in range(P))
            Gl, Ml = G, M
    f, r = fitness_eq3(normT2, Gl, S[-1], Ml, A[-1])
    return dict(A=A, S=S, f=f, r=r)


def par_pp_approx_sweep_sim(T, st_full: PPState, A, P, normT2):
    """Alg. 4 on the 1-D grid: Local-PP-init on each slab (no
    communication), local first-order terms, Reduce-Scatter of M~, V on replicated small
    matrices.  Returns the M~^(n) list (global) for comparison with the sequential sweep."""
    N = T.ndim
    sN = T.shape[-1]
    rng = [synth.slab_range(sN, p, P) for p in range(P)]
    locs = []
    for lo, hi in rng:
        Ap = st_full.Ap[:-1] + [st_full.Ap[-1][lo:hi]]
        locs.append(pp_init(T[..., lo:hi], Ap))
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    Ms = []
    for n in range(N):
        G = gamma(S, n)
        dA = [A[i] - st_full.Ap[i] for i in range(N)]
        parts = [pp_first_order(st, dA[:-1] + [dA[-1][lo:hi]], n) for (lo, hi), st in zip(rng, locs)]
        Mt = sum(parts) if n < N - 1 else np.concatenate(parts)
        Mt = Mt + A[n] @ pp_second_order(A, dA, S, n)
        A[n] = solve(G, Mt)
        S[n] = gram(A[n])
        Ms.append(Mt)
    return dict(A=A, M=Ms)


# ---------------------------------------------------------------------------
# Alg. 3 / Alg. 4 on a general N-D processor grid I_1 x ... x I_N (P:419-456, P:468-479,
# P:596-632): processor x = (x_1..x_N) holds the block T[b_1(x_1), ..., b_N(x_N)] with
# b_n(k) = synth.slab_range(s_n, k, I_n), and the factor rows b_m(x_m) of every mode.
# ---------------------------------------------------------------------------

def grid_procs(grid):
    """Processor coordinates in row-major order (last grid mode fastest): rank -> (x_1..x_N)."""
    return list(itertools.product(*[range(g) for g in grid]))


def _blk(shape, grid, x):
    return [synth.slab_range(s, k, g) for s, k, g in zip(shape, x, grid)]


def par_als_sweep_grid_sim(T, A, grid, normT2=None):
    """One sweep of Alg. 3 on the grid: Local-MTTKRP of every block with its local factor rows
    (line 13); the local results of the processors in Proc-Slice(x_n) summed into rows b_n(x_n)
    (Reduce-Scatter, line 14); solve (line 15); S^(n) as the sum of the Grams of the I = ∏I_n row
    chunks of the Q distribution (All-Reduce, lines 16-17); fitness by Eq. 3 on M^(N)."""
    N = T.ndim
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    if normT2 is None:
        normT2 = norm2(T)
    procs = grid_procs(grid)
    I = len(procs)
    for n in range(N):
        G = gamma(S, n)
        M = np.zeros((T.shape[n], A[0].shape[1]))
        for x in procs:
            b = _blk(T.shape, grid, x)
            Tx = T[tuple(slice(lo, hi) for lo, hi in b)]
            Ax = [A[m][lo:hi] for m, (lo, hi) in enumerate(b)]
            M[b[n][0]:b[n][1]] += mttkrp(Tx, Ax, n)
        A[n] = solve(G, M)
        # the Q distribution: ceil(s_n / I) rows per processor (line 5), the last chunks shorter
        c = -(-T.shape[n] // I)
        S[n] = sum(gram(A[n][q * c:(q + 1) * c]) for q in range(I) if q * c < T.shape[n])
        Gl, Ml = G, M
    f, r = fitness_eq3(normT2, Gl, S[-1], Ml, A[-1])
    return dict(A=A, S=S, f=f, r=r, M_last=Ml)


def par_pp_approx_sweep_grid_sim(T, st_full: PPState, A, grid, normT2):
    """Alg. 4 on the grid: Local-PP-init of every block with its local A_p rows (line 2, no
    communication), local first-order terms with the local dA rows (lines 5-7), M~^(n) summed over
    Proc-Slice(x_n) (line 9), V^(n) on the full small matrices (line 10).  Returns the M~^(n) list."""
    N = T.ndim
    procs = grid_procs(grid)
    blocks = [_blk(T.shape, grid, x) for x in procs]
    locs = [pp_init(T[tuple(slice(lo, hi) for lo, hi in b)], [st_full.Ap[m][lo:hi] for m, (lo, hi) in enumerate(b)])
            for b in blocks]
    A = [a.copy() for a in A]
    S = [gram(a) for a in A]
    Ms = []
    for n in range(N):
        G = gamma(S, n)
        dA = [A[i] - st_full.Ap[i] for i in range(N)]
        Mt = np.zeros((T.shape[n], A[0].shape[1]))
        for b, st in zip(blocks, locs):
            Mt[b[n][0]:b[n][1]] += pp_first_order(st, [dA[m][lo:hi] for m, (lo, hi) in enumerate(b)], n)
        Mt = Mt + A[n] @ pp_second_order(A, dA, S, n)
        A[n] = solve(G, Mt)
        S[n] = gram(A[n])
        Ms.append(Mt)
    return dict(A=A, M=Ms)
