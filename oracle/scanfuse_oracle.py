"""NumPy restatement of the reference pose solver (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/scanfuse/solver.py, frames.py:154-188,
geometry.py:40-186 and interp.py:8-58 operation for operation where the
rounding matters (frame-pair filter, association gates) and algebraically
elsewhere.  Poses are (R, t) tuples of float64 arrays; frames are objects
with the CachedFrame attributes; correspondence sets expose frame_i,
frame_j, points_i, points_j.

Single-threaded by design (the reference is single-threaded NumPy); the
bench's CPU baseline parallelises over processes at the edge level.
"""

from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------
# rigid-body helpers (geometry.py:40-186) on (R, t) tuples


def pose_of(p):
    return np.asarray(p.rotation, dtype=np.float64), np.asarray(p.translation, dtype=np.float64)


def inv(T):
    """geometry.py:144-146 — NumPy evaluates (-R.T) @ t."""
    Rt = T[0].T
    return Rt.copy(), -Rt @ T[1]


def compose(A, B):
    """geometry.py:127-130."""
    return A[0] @ B[0], A[0] @ B[1] + A[1]


def apply(T, pts):
    """geometry.py:148-151: pts @ R.T + t."""
    return np.asarray(pts, dtype=np.float64) @ T[0].T + T[1]


def cross_mat(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def exp_se3(xi):
    """exp_twist_vector (geometry.py:183-186) with so3_exp (:40-48) and the
    left Jacobian (:78-90), including both series branches."""
    w = np.asarray(xi[:3], dtype=np.float64)
    v = np.asarray(xi[3:6], dtype=np.float64)
    th = np.linalg.norm(w)
    K = cross_mat(w)
    if th < 1e-8:
        R = np.eye(3) + K + 0.5 * (K @ K)
    else:
        Kn = K / th
        R = np.eye(3) + np.sin(th) * Kn + (1.0 - np.cos(th)) * (Kn @ Kn)
    K2 = K @ K
    t2 = th * th
    if th < 1e-4:
        V = np.eye(3) + (0.5 - t2 / 24.0) * K + (1.0 / 6.0 - t2 / 120.0) * K2
    else:
        V = np.eye(3) + ((1.0 - np.cos(th)) / t2) * K + ((th - np.sin(th)) / (t2 * th)) * K2
    return R, V @ v


def project(k, q):
    """Intrinsics.project_many (geometry.py:219-227)."""
    z = q[:, 2]
    front = z > 0.0
    zs = np.where(front, z, 1.0)
    return k.fx * q[:, 0] / zs + k.cx, k.fy * q[:, 1] / zs + k.cy, front


def inside_cont(k, u, v, front):
    return front & (u >= 0.0) & (u <= k.width - 1) & (v >= 0.0) & (v <= k.height - 1)


# --------------------------------------------------------------------------
# pair filter (solver.py:130-148, frames.py:154-188)


def view_angle_deg(Ta, Tb) -> float:
    c = np.clip(np.dot(Ta[0][:, 2], Tb[0][:, 2]), -1.0, 1.0)
    return float(np.degrees(np.arccos(c)))


def frustum_overlap(ca, Ta, cb, Tb) -> float:
    vd = ca.valid_depth
    if not np.any(vd):
        return 0.0
    pts = ca.points_low[vd].astype(np.float64)
    rel = compose(inv(Tb), Ta)
    u, v, f = project(cb.intrinsics_low, apply(rel, pts))
    return float(np.count_nonzero(inside_cont(cb.intrinsics_low, u, v, f))) / float(pts.shape[0])


def dense_edges(ids, poses, caches, max_deg=60.0):
    out = []
    for a in range(len(ids)):
        for b in range(a + 1, len(ids)):
            i, j = ids[a], ids[b]
            if view_angle_deg(poses[i], poses[j]) >= max_deg:
                continue
            if frustum_overlap(caches[i], poses[i], caches[j], poses[j]) <= 0.0:
                continue
            if frustum_overlap(caches[j], poses[j], caches[i], poses[i]) <= 0.0:
                continue
            out.append((i, j))
    return out


# --------------------------------------------------------------------------
# dense terms (solver.py:158-328, interp.py:8-58)


def source_pixels(c, stride, geo):
    m = c.valid_depth.copy()
    if geo:
        m &= c.valid_normal
    if stride > 1:
        g = np.zeros_like(m)
        g[::stride, ::stride] = True
        m &= g
    return np.nonzero(m)


def assoc_photo(poses, i, j, ci, cj, stride=1):
    """-> (points (m,3), reference (m,2)) (solver.py:216-232)."""
    ys, xs = source_pixels(ci, stride, False)
    pts = ci.points_low[ys, xs].astype(np.float64)
    ref = ci.grad_low[ys, xs].astype(np.float64)
    rel = compose(inv(poses[j]), poses[i])
    u, v, f = project(cj.intrinsics_low, apply(rel, pts))
    keep = inside_cont(cj.intrinsics_low, u, v, f)
    return pts[keep], ref[keep]


def assoc_geo(poses, i, j, ci, cj, dmax=0.15, nmin=0.9, stride=1):
    """-> (points, normals, targets) (solver.py:235-260)."""
    ys, xs = source_pixels(ci, stride, True)
    pts = ci.points_low[ys, xs].astype(np.float64)
    nrm = ci.normals_low[ys, xs].astype(np.float64)
    rel = compose(inv(poses[j]), poses[i])
    q = apply(rel, pts)
    k = cj.intrinsics_low
    u, v, f = project(k, q)
    xi = np.round(u).astype(int)
    yi = np.round(v).astype(int)
    ok = f & (xi >= 0) & (xi < k.width) & (yi >= 0) & (yi < k.height)
    xi = np.clip(xi, 0, k.width - 1)
    yi = np.clip(yi, 0, k.height - 1)
    tok = cj.valid_depth[yi, xi] & cj.valid_normal[yi, xi]
    tgt = cj.points_low[yi, xi].astype(np.float64)
    tn = cj.normals_low[yi, xi].astype(np.float64)
    dist = np.linalg.norm(q - tgt, axis=1)
    ndot = np.sum((nrm @ rel[0].T) * tn, axis=1)
    keep = ok & tok & (dist < dmax) & (ndot > nmin)
    return pts[keep], nrm[keep], tgt[keep]


def bilinear2(img, x, y):
    """bilinear_sample_with_grad (interp.py:36-58) for an (H,W,C) image."""
    h, w = img.shape[:2]
    x = np.clip(x, 0.0, w - 1.0)
    y = np.clip(y, 0.0, h - 1.0)
    x0 = np.minimum(np.floor(x), w - 2).astype(int)
    y0 = np.minimum(np.floor(y), h - 2).astype(int)
    ax = (x - x0)[:, None]
    ay = (y - y0)[:, None]
    a, b = img[y0, x0], img[y0, x0 + 1]
    c, d = img[y0 + 1, x0], img[y0 + 1, x0 + 1]
    val = a * (1 - ax) * (1 - ay) + b * ax * (1 - ay) + c * (1 - ax) * ay + d * ax * ay
    gx = (b - a) * (1 - ay) + (d - c) * ay
    gy = (c - a) * (1 - ax) + (d - b) * ax
    return val, gx, gy


def photo_res(poses, i, j, pts, ref, cj):
    """solver.py:263-274."""
    if pts.shape[0] == 0:
        return np.zeros((0, 2))
    rel = compose(inv(poses[j]), poses[i])
    u, v, _ = project(cj.intrinsics_low, apply(rel, pts))
    val, _, _ = bilinear2(cj.grad_low.astype(np.float64), u, v)
    return ref - val


def geo_res(poses, i, j, pts, nrm, tgt):
    """solver.py:277-283."""
    if pts.shape[0] == 0:
        return np.zeros(0)
    back = compose(inv(poses[i]), poses[j])
    return np.sum(nrm * (pts - apply(back, tgt)), axis=1)


def photo_lin(poses, i, j, pts, ref, cj):
    """solver.py:286-310 -> (res (m,2), J_i (m,2,6)); J_j = -J_i."""
    m = pts.shape[0]
    if m == 0:
        return np.zeros((0, 2)), np.zeros((0, 2, 6))
    Ti, Tj = poses[i], poses[j]
    wld = apply(Ti, pts)
    q = apply(inv(Tj), wld)
    k = cj.intrinsics_low
    u, v, _ = project(k, q)
    val, gx, gy = bilinear2(cj.grad_low.astype(np.float64), u, v)
    z = q[:, 2]
    # d(value)/dq per channel: [gx fx/z, gy fy/z, -(gx fx x + gy fy y)/z^2]
    dq = np.stack([gx * (k.fx / z)[:, None], gy * (k.fy / z)[:, None],
                   -(gx * (k.fx * q[:, 0] / z ** 2)[:, None] + gy * (k.fy * q[:, 1] / z ** 2)[:, None])],
                  axis=2)                                   # (m, 2, 3)
    g = dq @ Tj[0].T                                        # dval/dq R_j^T (solver.py:308)
    J = np.empty((m, 2, 6))
    J[:, :, :3] = np.cross(g, wld[:, None, :])
    J[:, :, 3:] = -g
    return ref - val, J


def geo_lin(poses, i, j, pts, nrm, tgt):
    """solver.py:313-328 -> (res (m,), J_i (m,6)); J_j = -J_i."""
    if pts.shape[0] == 0:
        return np.zeros(0), np.zeros((0, 6))
    Ti, Tj = poses[i], poses[j]
    wt = apply(Tj, tgt)
    mapped = apply(inv(Ti), wt)
    res = np.sum(nrm * (pts - mapped), axis=1)
    mvec = nrm @ Ti[0].T
    J = np.concatenate([np.cross(wt, mvec), mvec], axis=1)
    return res, J


# --------------------------------------------------------------------------
# system (solver.py:356-454, 568-660)


class System:
    """Sparse matrix-free part + dense n_vars^2 part, like NormalEquations."""

    def __init__(self, n_vars, w_s, yi, yj, vi, vj, grad, dense=None):
        self.n_vars, self.w_s = n_vars, w_s
        self.yi, self.yj, self.vi, self.vj = yi, yj, vi, vj
        self.gradient = grad
        self.dense = dense
        self.diagonal = self._diag()

    @property
    def rhs(self):
        return -self.gradient

    def _scatter(self, w):
        """J^T w (solver.py:389-401)."""
        out = np.zeros((self.n_vars // 6, 6))
        for var, y, s in ((self.vi, self.yi, 1.0), (self.vj, self.yj, -1.0)):
            a = var >= 0
            if np.any(a):
                np.add.at(out, var[a], s * np.concatenate([np.cross(y[a], w[a]), w[a]], axis=1))
        return out.ravel()

    def _gather(self, x):
        """J x (solver.py:375-387)."""
        blk = x.reshape(-1, 6)
        out = np.zeros((self.yi.shape[0], 3))
        for var, y, s in ((self.vi, self.yi, 1.0), (self.vj, self.yj, -1.0)):
            a = var >= 0
            if np.any(a):
                g = blk[var[a]]
                out[a] += s * (g[:, 3:] + np.cross(g[:, :3], y[a]))
        return out

    def apply(self, x):
        out = np.zeros(self.n_vars)
        if self.yi.shape[0] and self.w_s > 0.0:
            out += self.w_s * self._scatter(self._gather(x))
        if self.dense is not None:
            out += self.dense @ x
        return out

    def _diag(self):
        d = np.zeros((self.n_vars // 6, 6))
        if self.yi.shape[0] and self.w_s > 0.0:
            for var, y in ((self.vi, self.yi), (self.vj, self.yj)):
                a = var >= 0
                if np.any(a):
                    yy = y[a] ** 2
                    c = np.concatenate([yy.sum(axis=1)[:, None] - yy, np.ones((yy.shape[0], 3))], axis=1)
                    np.add.at(d, var[a], self.w_s * c)
        d = d.ravel()
        if self.dense is not None:
            d = d + np.diag(self.dense)
        return d

    def materialize(self):
        cols = [self.apply(e) for e in np.eye(self.n_vars)]
        return np.stack(cols, axis=1) if cols else np.zeros((0, 0))


class Problem:
    """Oracle state for one solve: frames in order, poses, stacked sparse term."""

    def __init__(self, ids, poses, sets, caches=None):
        self.ids = list(ids)
        self.poses = {f: pose_of(poses[f]) if not isinstance(poses[f], tuple) else poses[f]
                      for f in self.ids}
        self.sets = list(sets)
        self.caches = caches
        self.var = {f: k - 1 for k, f in enumerate(self.ids)}
        self.n_vars = 6 * (len(self.ids) - 1)
        if self.sets:
            self.fi = np.concatenate([np.full(len(s), s.frame_i) for s in self.sets])
            self.fj = np.concatenate([np.full(len(s), s.frame_j) for s in self.sets])
            self.pi = np.vstack([np.asarray(s.points_i, float) for s in self.sets])
            self.pj = np.vstack([np.asarray(s.points_j, float) for s in self.sets])
        else:
            self.fi = self.fj = np.zeros(0, dtype=int)
            self.pi = self.pj = np.zeros((0, 3))
        self.vi = np.array([self.var[f] for f in self.fi], dtype=int)
        self.vj = np.array([self.var[f] for f in self.fj], dtype=int)
        self.edges = []

    def world(self):
        """_sparse_state (solver.py:568-580)."""
        if not self.sets:
            return np.zeros((0, 3)), np.zeros((0, 3))
        Ri = np.stack([self.poses[f][0] for f in self.fi])
        Rj = np.stack([self.poses[f][0] for f in self.fj])
        ti = np.stack([self.poses[f][1] for f in self.fi])
        tj = np.stack([self.poses[f][1] for f in self.fj])
        return (np.einsum("nab,nb->na", Ri, self.pi) + ti,
                np.einsum("nab,nb->na", Rj, self.pj) + tj)

    def directed(self, bidir):
        d = list(self.edges)
        if bidir:
            d += [(j, i) for (i, j) in self.edges]
        return d

    def linearize(self, w, w_dense, cfg):
        """normal_equations (solver.py:630-660) + _dense_blocks (:582-628).

        Returns (System, energy, frozen) with frozen = (photo list, geo list)."""
        yi, yj = self.world()
        r = yi - yj
        proto = System(self.n_vars, w["sparse"], yi, yj, self.vi, self.vj, np.zeros(self.n_vars))
        grad = np.zeros(self.n_vars)
        if r.shape[0]:
            grad += w["sparse"] * proto._scatter(r)
        energy = w["sparse"] * float(np.sum(r ** 2))
        dense = None
        frozen = ([], [])
        if self.caches is not None and w_dense > 0.0 and self.edges:
            dense = np.zeros((self.n_vars, self.n_vars))
            ep = eg = 0.0
            st = cfg.get("dense_pixel_stride", 1)
            for (i, j) in self.directed(cfg.get("dense_bidirectional", False)):
                ci, cj = self.caches[i], self.caches[j]
                a, b = self.var[i], self.var[j]
                if w["photo"] > 0.0:
                    pts, ref = assoc_photo(self.poses, i, j, ci, cj, st)
                    frozen[0].append((i, j, pts, ref))
                    if pts.shape[0]:
                        res, J = photo_lin(self.poses, i, j, pts, ref, cj)
                        ep += float(np.sum(res ** 2))
                        self._acc(dense, grad, J.reshape(-1, 6), res.reshape(-1), a, b,
                                  w_dense * w["photo"])
                if w["geo"] > 0.0:
                    pts, nrm, tgt = assoc_geo(self.poses, i, j, ci, cj, cfg.get("geo_distance_max", 0.15),
                                              cfg.get("geo_normal_min", 0.9), st)
                    frozen[1].append((i, j, pts, nrm, tgt))
                    if pts.shape[0]:
                        res, J = geo_lin(self.poses, i, j, pts, nrm, tgt)
                        self._acc(dense, grad, J, res, a, b, w_dense * w["geo"])
                        eg += float(np.sum(res ** 2))
            energy += w_dense * (w["photo"] * ep + w["geo"] * eg)
        return System(self.n_vars, w["sparse"], yi, yj, self.vi, self.vj, grad, dense), energy, frozen

    @staticmethod
    def _acc(A, g, J, res, a, b, s):
        """_accumulate (solver.py:615-628) with J_j = -J_i."""
        H = s * (J.T @ J)
        gi = s * (J.T @ res)
        for va, sa in ((a, 1.0), (b, -1.0)):
            if va < 0:
                continue
            g[6 * va:6 * va + 6] += sa * gi
            for vb, sb in ((a, 1.0), (b, -1.0)):
                if vb >= 0:
                    A[6 * va:6 * va + 6, 6 * vb:6 * vb + 6] += sa * sb * H

    def frozen_energy(self, w, w_dense, frozen):
        """_energy_with_frozen_associations (solver.py:662-672)."""
        yi, yj = self.world_apply()
        e = w["sparse"] * float(np.sum((yi - yj) ** 2))
        if w_dense > 0.0:
            ep = sum(float(np.sum(photo_res(self.poses, i, j, p, rf, self.caches[j]) ** 2))
                     for (i, j, p, rf) in frozen[0])
            eg = sum(float(np.sum(geo_res(self.poses, i, j, p, n, t) ** 2))
                     for (i, j, p, n, t) in frozen[1])
            e += w_dense * (w["photo"] * ep + w["geo"] * eg)
        return e

    def world_apply(self):
        """eval_sparse's RigidTransform.apply path (solver.py:114-123)."""
        if not self.sets:
            return np.zeros((0, 3)), np.zeros((0, 3))
        yi = np.vstack([apply(self.poses[s.frame_i], s.points_i) for s in self.sets])
        yj = np.vstack([apply(self.poses[s.frame_j], s.points_j) for s in self.sets])
        return yi, yj

    def step(self, dx):
        """_apply_step (solver.py:674-677)."""
        for f in self.ids[1:]:
            k = self.var[f]
            self.poses[f] = compose(exp_se3(dx[6 * k:6 * k + 6]), self.poses[f])


def pcg(sys, max_it=50, tol=1e-6, restart=20):
    """pcg_solve (solver.py:463-508): -> (x, iterations, relative, diverged)."""
    b = sys.rhs
    nb = np.linalg.norm(b)
    x = np.zeros_like(b)
    if nb == 0.0:
        return x, 0, 0.0, False
    inv_d = 1.0 / np.maximum(sys.diagonal, 1e-12)
    r = b.copy()
    z = inv_d * r
    p = z.copy()
    rz = float(r @ z)
    rel, its = 1.0, 0
    for k in range(1, max_it + 1):
        its = k
        Ap = sys.apply(p)
        pAp = float(p @ Ap)
        if not np.isfinite(pAp):
            return x, its, rel, True
        if pAp <= 0.0:
            break
        a = rz / pAp
        x += a * p
        r = b - sys.apply(x) if k % restart == 0 else r - a * Ap
        if not np.all(np.isfinite(x)):
            return x, its, rel, True
        rel = float(np.linalg.norm(r) / nb)
        if rel < tol:
            break
        z = inv_d * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, its, rel, False


def ramp(w, it):
    """dense_ramp_weight (solver.py:49-53)."""
    s, e = w.get("dense_ramp", (0, 5))
    if e <= s:
        return 1.0 if it >= e else 0.0
    return float(np.clip((it - s) / (e - s), 0.0, 1.0))


DEFAULT_W = dict(sparse=1.0, photo=0.1, geo=1.0, dense_ramp=(0, 5))
DEFAULT_CFG = dict(batch_iterations=10, pcg_max_iterations=50, pcg_tolerance=1e-6,
                   pcg_restart_interval=20, min_relative_decrease=1e-9, view_angle_max_deg=60.0,
                   geo_distance_max=0.15, geo_normal_min=0.9, dense_pixel_stride=1,
                   dense_bidirectional=False, prune_residual_max=0.05)


def solve(ids, poses, sets, caches=None, weights=None, config=None, max_iterations=None):
    """AlignmentProblem.solve (solver.py:681-750).

    Returns (final poses dict of (R,t), records list of dicts, converged, aborted, edges)."""
    w = dict(DEFAULT_W, **(weights or {}))
    cfg = dict(DEFAULT_CFG, **(config or {}))
    if max_iterations is None:
        max_iterations = cfg["batch_iterations"]
    P = Problem(ids, poses, sets, caches)
    recs, conv, abort = [], False, False
    if P.n_vars == 0:
        return P.poses, recs, True, False, []
    if caches is not None:
        P.edges = dense_edges(P.ids, P.poses, caches, cfg["view_angle_max_deg"])
    best_e, best = np.inf, dict(P.poses)
    inc = 0
    for it in range(max_iterations):
        wd = ramp(w, it)
        S, e0, frozen = P.linearize(w, wd, cfg)
        if e0 <= 1e-18:
            conv = True
            recs.append(dict(iteration=it, energy_before=e0, energy_after=e0, dense_weight=wd,
                             pcg_iterations=0, pcg_residual=0.0, step_norm=0.0, accepted=True))
            break
        dx, its, rel, bad = pcg(S, cfg["pcg_max_iterations"], cfg["pcg_tolerance"],
                                cfg["pcg_restart_interval"])
        if bad:
            abort = True
            break
        P.step(dx)
        e1 = P.frozen_energy(w, wd, frozen)
        acc = e1 <= e0
        recs.append(dict(iteration=it, energy_before=e0, energy_after=e1, dense_weight=wd,
                         pcg_iterations=its, pcg_residual=rel, step_norm=float(np.linalg.norm(dx)),
                         accepted=acc))
        if acc:
            inc = 0
        else:
            inc += 1
            if inc >= 2:
                P.poses = best
                abort = True
                break
        if e1 < best_e:
            best_e, best = e1, dict(P.poses)
        if acc and (e0 - e1) < cfg["min_relative_decrease"] * max(e0, 1e-30):
            conv = True
            break
    else:
        conv = True
    return P.poses, recs, conv, abort, P.edges


def max_residual_set(poses, sets):
    """solver.py:765-776."""
    worst_set, worst = -1, -1.0
    for idx, cs in enumerate(sets):
        Ti = poses[cs.frame_i] if isinstance(poses[cs.frame_i], tuple) else pose_of(poses[cs.frame_i])
        Tj = poses[cs.frame_j] if isinstance(poses[cs.frame_j], tuple) else pose_of(poses[cs.frame_j])
        res = np.linalg.norm(apply(Ti, cs.points_i) - apply(Tj, cs.points_j), axis=1)
        peak = float(res.max()) if res.size else 0.0
        if peak > worst:
            worst, worst_set = peak, idx
    return worst_set, worst


# --------------------------------------------------------------------------
# dense_verify (filters.py:200-277)


def bilinear1(img, x, y):
    """bilinear_sample (interp.py:17-33) of a single-channel image, with
    _corner_indices (interp.py:8-14); NumPy evaluation order."""
    img = np.asarray(img)
    h, w = img.shape[:2]
    x = np.clip(np.asarray(x, float), 0.0, w - 1.0)
    y = np.clip(np.asarray(y, float), 0.0, h - 1.0)
    x0 = np.minimum(np.floor(x), w - 2).astype(int)
    y0 = np.minimum(np.floor(y), h - 2).astype(int)
    fx, fy = x - x0, y - y0
    return (img[y0, x0] * (1 - fx) * (1 - fy) + img[y0, x0 + 1] * fx * (1 - fy)
            + img[y0 + 1, x0] * (1 - fx) * fy + img[y0 + 1, x0 + 1] * fx * fy)


def verify_one_direction(src, dst, T, depth_max=0.15, normal_min=0.9, color_max=0.1):
    """_verify_one_direction (filters.py:216-250): (mean_error, count).
    T = (R, t) maps src camera space into dst camera space."""
    eligible = src.valid_depth & src.valid_normal
    if not np.any(eligible):
        return 0.0, 0
    pts = src.points_low[eligible].astype(np.float64)
    nrm = src.normals_low[eligible].astype(np.float64)
    inten = src.intensity_low[eligible].astype(np.float64)
    moved = pts @ T[0].T + T[1]
    k = dst.intrinsics_low
    u, v, front = project(k, moved)
    xi = np.round(u).astype(int)
    yi = np.round(v).astype(int)
    inside = front & (xi >= 0) & (xi < k.width) & (yi >= 0) & (yi < k.height)
    xi, yi = np.clip(xi, 0, k.width - 1), np.clip(yi, 0, k.height - 1)
    ok = dst.valid_depth[yi, xi] & dst.valid_normal[yi, xi] & inside
    dist = np.linalg.norm(moved - dst.points_low[yi, xi].astype(np.float64), axis=1)
    ndot = np.sum((nrm @ T[0].T) * dst.normals_low[yi, xi].astype(np.float64), axis=1)
    cdiff = np.abs(inten - bilinear1(dst.intensity_low, u, v))
    good = ok & (dist < depth_max) & (ndot > normal_min) & (cdiff < color_max)
    count = int(np.count_nonzero(good))
    return (float(dist[good].sum() / count) if count else 0.0), count


def dense_verify(ci, cj, T, depth_max=0.15, normal_min=0.9, color_max=0.1, error_max=0.075,
                 min_fraction=0.02):
    """dense_verify (filters.py:253-277): (passed, err_ij, err_ji, count_ij, count_ji)."""
    e1, n1 = verify_one_direction(ci, cj, T, depth_max, normal_min, color_max)
    e2, n2 = verify_one_direction(cj, ci, inv(T), depth_max, normal_min, color_max)
    k = ci.intrinsics_low
    m = min_fraction * k.width * k.height
    return (n1 >= m and n2 >= m and e1 <= error_max and e2 <= error_max), e1, e2, n1, n2


# --------------------------------------------------------------------------
# hashed TSDF integrate / de-integrate (tsdf.py:55-201)

TSDF_B = 8  # voxels per block edge (tsdf.py:21)


def _block_offsets():
    i, j, k = np.meshgrid(np.arange(TSDF_B), np.arange(TSDF_B), np.arange(TSDF_B), indexing="ij")
    return np.stack([i, j, k], axis=-1).reshape(-1, 3).astype(np.float64)


class TsdfOracle:
    """TsdfVolume restated: blocks = {coord: [weight, wdist, wcolor]} (float32
    accumulators, insertion order = allocation order).  integrate/deintegrate
    follow tsdf.py:90-160 step for step; errors raise ValueError."""

    EPS = np.float32(1e-6)

    def __init__(self, voxel_size=0.004, truncation=None, depth_weighting=False):
        self.vs = float(voxel_size)
        self.trunc = float(truncation if truncation is not None else max(0.02, 5.0 * voxel_size))
        self.dw = depth_weighting
        self.blocks = {}

    @property
    def extent(self):
        return self.vs * TSDF_B

    def touched(self, depth_img, K, T):
        """tsdf.py:162-181: sorted unique block coords the truncation band crosses."""
        valid = depth_img > 0.0
        if not np.any(valid):
            return np.zeros((0, 3), dtype=np.int64)
        ys, xs = np.nonzero(valid)
        d = depth_img[ys, xs].astype(np.float64)
        rays = np.stack([(xs.astype(np.float64) - K.cx) / K.fx * 1.0,
                         (ys.astype(np.float64) - K.cy) / K.fy * 1.0, np.ones_like(d)], axis=-1)
        wn = apply(T, rays * np.maximum(d - self.trunc, 1e-3)[:, None])
        wf = apply(T, rays * (d + self.trunc)[:, None])
        n = max(2, int(np.ceil(4.0 * self.trunc / self.extent)) + 1)
        keys = set()
        allk = []
        for s in np.linspace(0.0, 1.0, n):
            c = np.floor((wn + s * (wf - wn)) / self.extent).astype(np.int64)
            allk.append(c)
        c = np.unique(np.concatenate(allk), axis=0)
        del keys
        return c  # np.unique(axis=0) sorts lexicographically == the packed-key order

    def apply_frame(self, color, depth_img, K, T, sign):
        tb = self.touched(depth_img, K, T)
        if tb.shape[0] == 0:
            if sign < 0:
                raise ValueError("frame has no integrated content")
            return
        cen = (tb[:, None, :] * self.extent + (_block_offsets()[None] + 0.5) * self.vs).reshape(-1, 3)
        cam = apply(inv(T), cen)
        u, v, front = project(K, cam)
        xi, yi = np.round(u).astype(int), np.round(v).astype(int)
        ins = front & (xi >= 0) & (xi < K.width) & (yi >= 0) & (yi < K.height)
        xi, yi = np.clip(xi, 0, K.width - 1), np.clip(yi, 0, K.height - 1)
        d = depth_img[yi, xi].astype(np.float64)
        sdf = d - cam[:, 2]
        hit = (ins & (d > 0.0) & (np.abs(sdf) <= self.trunc)).reshape(-1, 512)
        if self.dw:
            wgt = np.where(cam[:, 2] > 0.0, 1.0 / np.maximum(cam[:, 2], 1e-6), 0.0)
        else:
            wgt = np.ones_like(sdf)
        col = color[yi, xi].astype(np.float64)
        wd = (wgt * sdf).reshape(-1, 512).astype(np.float32)
        w = wgt.reshape(-1, 512).astype(np.float32)
        wc = (wgt[:, None] * col).reshape(-1, 512, 3).astype(np.float32)
        s = np.float32(sign)
        for b, key in enumerate(map(tuple, tb.tolist())):
            h = hit[b]
            blk = self.blocks.get(key)
            if not h.any():
                if sign < 0 and blk is not None and not blk[0].any():
                    del self.blocks[key]
                continue
            if blk is None:
                if sign < 0:
                    raise ValueError(f"block {key} missing")
                blk = [np.zeros(512, np.float32), np.zeros(512, np.float32),
                       np.zeros((512, 3), np.float32)]
                self.blocks[key] = blk
            blk[0][h] += s * w[b][h]
            blk[1][h] += s * wd[b][h]
            blk[2][h] += s * wc[b][h]
            if sign < 0:
                if (blk[0] < -self.EPS).any():
                    raise ValueError(f"negative weight in block {key}")
                snap = (np.abs(blk[0]) <= self.EPS) & (blk[0] != 0.0)
                blk[0][snap] = 0.0
                z = blk[0] == 0.0
                blk[1][z] = 0.0
                blk[2][z] = 0.0
                if not blk[0].any():
                    del self.blocks[key]
