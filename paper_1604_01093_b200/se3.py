"""Host-side pose and camera records (the data formats either side of the solver).

These mirror the attribute layout of the reference's `scanfuse.geometry`
records (`RigidTransform` geometry.py:104-153, `TwistParams` :158-175,
`Intrinsics` :197-249) so the drop-in solver accepts either the reference's
objects or these; the solver itself only reads `.rotation`, `.translation`
and the intrinsics fields.  Poses map camera coordinates into the parent
frame, T(p) = R p + t; twists are (omega, v) composed on the left.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SMALL_ANGLE = 1e-8      # geometry.py:24 (so3 series branch)
SERIES_ANGLE = 1e-4     # geometry.py:75 (left-Jacobian series branch)


def skew(v) -> np.ndarray:
    """Cross-product matrix [v]x."""
    a, b, c = (float(x) for x in v)
    return np.array([[0.0, -c, b], [c, 0.0, -a], [-b, a, 0.0]])


def so3_exp(omega) -> np.ndarray:
    """Rodrigues' formula; second-order series below SMALL_ANGLE."""
    w = np.asarray(omega, dtype=np.float64)
    theta = np.linalg.norm(w)
    K = skew(w)
    if theta < SMALL_ANGLE:
        return np.eye(3) + K + 0.5 * (K @ K)
    Kn = K / theta
    return np.eye(3) + np.sin(theta) * Kn + (1.0 - np.cos(theta)) * (Kn @ Kn)


def left_jacobian(omega) -> np.ndarray:
    """V(omega) of the SE(3) exponential."""
    w = np.asarray(omega, dtype=np.float64)
    theta = np.linalg.norm(w)
    K = skew(w)
    K2 = K @ K
    t2 = theta * theta
    if theta < SERIES_ANGLE:
        c1, c2 = 0.5 - t2 / 24.0, 1.0 / 6.0 - t2 / 120.0
    else:
        c1, c2 = (1.0 - np.cos(theta)) / t2, (theta - np.sin(theta)) / (t2 * theta)
    return np.eye(3) + c1 * K + c2 * K2


@dataclass
class RigidTransform:
    rotation: np.ndarray
    translation: np.ndarray

    @classmethod
    def identity(cls) -> "RigidTransform":
        return cls(np.eye(3), np.zeros(3))

    @classmethod
    def from_matrix(cls, m) -> "RigidTransform":
        m = np.asarray(m, dtype=np.float64)
        return cls(m[:3, :3].copy(), m[:3, 3].copy())

    def matrix(self) -> np.ndarray:
        out = np.eye(4)
        out[:3, :3], out[:3, 3] = self.rotation, self.translation
        return out

    def compose(self, other: "RigidTransform") -> "RigidTransform":
        R = self.rotation
        return RigidTransform(R @ other.rotation, R @ other.translation + self.translation)

    __matmul__ = compose

    def inverse(self) -> "RigidTransform":
        Rt = self.rotation.T
        return RigidTransform(Rt.copy(), -Rt @ self.translation)

    def apply(self, points) -> np.ndarray:
        return np.asarray(points, dtype=np.float64) @ self.rotation.T + self.translation

    def rotate(self, vectors) -> np.ndarray:
        return np.asarray(vectors, dtype=np.float64) @ self.rotation.T


@dataclass
class TwistParams:
    omega: np.ndarray
    v: np.ndarray

    def as_vector(self) -> np.ndarray:
        return np.concatenate([self.omega, self.v])


def exp_twist(xi: TwistParams) -> RigidTransform:
    w = np.asarray(xi.omega, dtype=np.float64)
    return RigidTransform(so3_exp(w), left_jacobian(w) @ np.asarray(xi.v, dtype=np.float64))


def exp_twist_vector(xi6) -> RigidTransform:
    x = np.asarray(xi6, dtype=np.float64)
    return RigidTransform(so3_exp(x[:3]), left_jacobian(x[:3]) @ x[3:6])


@dataclass
class Intrinsics:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def project_many(self, points):
        p = np.asarray(points, dtype=np.float64)
        z = p[..., 2]
        front = z > 0.0
        zs = np.where(front, z, 1.0)
        return np.stack([self.fx * p[..., 0] / zs + self.cx,
                         self.fy * p[..., 1] / zs + self.cy], axis=-1), front

    def unproject(self, pixel, depth):
        pixel = np.asarray(pixel, dtype=np.float64)
        depth = np.asarray(depth, dtype=np.float64)
        return np.stack([(pixel[..., 0] - self.cx) / self.fx * depth,
                         (pixel[..., 1] - self.cy) / self.fy * depth, depth], axis=-1)

    def scaled(self, new_width: int, new_height: int) -> "Intrinsics":
        sx, sy = new_width / self.width, new_height / self.height
        return Intrinsics(self.fx * sx, self.fy * sy, (self.cx + 0.5) * sx - 0.5,
                          (self.cy + 0.5) * sy - 0.5, new_width, new_height)
