"""TEST INFRASTRUCTURE: restatements of the reference's own test oracles
(proj/tests/oracles.hpp) and of the operators they use (solver.cpp:53-101),
in numpy, for the acceptance criteria run against the GPU stepper. Never
imported by the product.

  dense_radial_half_step / dense_axial_half_step  oracles.hpp:61-176
  apply_lambda_r / apply_lambda_z                 solver.cpp:53-101
  face_lambda                                     materials.hpp:101-124
"""
from __future__ import annotations

import math

import numpy as np

from paper_1912_03744_b200.materials import HalfPointRule, Property


def face_lambda(own, other, a, b, cfg):  # materials.hpp:101-124
    pol = cfg.range_policy
    if cfg.halfpoint_rule == HalfPointRule.MeanLambda:
        return 0.5 * (own.eval(Property.Conductivity, a, pol) +
                      own.eval(Property.Conductivity, b, pol))
    if cfg.halfpoint_rule == HalfPointRule.TwoSidedHarmonic:
        la = own.eval(Property.Conductivity, a, pol)
        lb = other.eval(Property.Conductivity, b, pol)
        return 2.0 * la * lb / (la + lb)
    return own.eval(Property.Conductivity, 0.5 * (a + b), pol)


def apply_lambda_r(grid, mats, f, i, j, cfg):  # solver.cpp:53-75
    n = grid.row_extent(j)
    lo = hi = 0.0
    if i > 0:
        coef = grid.face_r_lo(i) * face_lambda(mats[grid.layer(i - 1)], mats[grid.layer(i)],
                                               f[i - 1, j], f[i, j], cfg) / grid.gap_r(i)
        lo = coef * (f[i, j] - f[i - 1, j])
    if i < n - 1:
        coef = grid.face_r_lo(i + 1) * face_lambda(mats[grid.layer(i)], mats[grid.layer(i + 1)],
                                                   f[i, j], f[i + 1, j], cfg) / grid.gap_r(i + 1)
        hi = coef * (f[i + 1, j] - f[i, j])
    return (hi - lo) / (grid.r_center(i) * grid.control_r(i))


def apply_lambda_z(grid, mats, f, i, j, cfg):  # solver.cpp:77-101
    m = grid.col_extent(i)
    mat = mats[grid.layer(i)]
    lo = hi = 0.0
    if j > 0:
        lo = face_lambda(mat, mat, f[i, j - 1], f[i, j], cfg) / grid.gap_z(j) * (f[i, j] - f[i, j - 1])
    if j < m - 1:
        hi = face_lambda(mat, mat, f[i, j], f[i, j + 1], cfg) / grid.gap_z(j + 1) * (f[i, j + 1] - f[i, j])
    elif grid.layer(i) == 0 and not cfg.all_neumann:
        lam = mat.eval(Property.Conductivity, cfg.T0, cfg.range_policy)
        hi = lam * (cfg.T0 - f[i, j]) / (0.5 * grid.width_z(j))
    return (hi - lo) / grid.control_z(j)


def joule_power(case, source, i, T):
    """JouleSource::power after bind_time (source.hpp:68-72)."""
    if i is None or source is None or source.pulse == 0.0:
        return 0.0
    mat = case.materials[case.domain.source_layer]
    return (mat.eval(Property.Resistivity, T, case.solver.range_policy) * source.amplitude) \
        * source.pulse


def _cells(grid):
    idx = {}
    for j in range(grid.nz()):
        for i in range(grid.row_extent(j)):
            idx[(i, j)] = len(idx)
    return idx


def dense_radial_half_step(case, source, T_cur, tau, stop_tol, max_sweeps=200):
    """oracles.hpp:61-115: the whole implicit-in-r system over the masked
    cells, coefficients frozen at the iterate, re-solved until it settles."""
    grid, mats, cfg = case.grid(), case.materials, case.solver
    idx = _cells(grid)
    it = T_cur.copy(order="F")
    for _ in range(max_sweeps):
        A = np.zeros((len(idx), len(idx)))
        rhs = np.zeros(len(idx))
        for j in range(grid.nz()):
            n = grid.row_extent(j)
            for i in range(n):
                row = idx[(i, j)]
                mat = mats[grid.layer(i)]
                vol = grid.r_center(i) * grid.control_r(i)
                K = mat.rho() * mat.eval(Property.HeatCapacity, it[i, j], cfg.range_policy) / (0.5 * tau)
                A[row, row] += K
                rhs[row] += K * T_cur[i, j]
                if i > 0:
                    c = grid.face_r_lo(i) * face_lambda(mats[grid.layer(i - 1)], mat, it[i - 1, j],
                                                        it[i, j], cfg) / (grid.gap_r(i) * vol)
                    A[row, row] += c
                    A[row, idx[(i - 1, j)]] -= c
                if i < n - 1:
                    c = grid.face_r_lo(i + 1) * face_lambda(mat, mats[grid.layer(i + 1)], it[i, j],
                                                            it[i + 1, j], cfg) / (grid.gap_r(i + 1) * vol)
                    A[row, row] += c
                    A[row, idx[(i + 1, j)]] -= c
                rhs[row] += apply_lambda_z(grid, mats, T_cur, i, j, cfg)
                rhs[row] += joule_power(case, source, i if grid.layer(i) == case.domain.source_layer
                                        else None, it[i, j])
        sol = np.linalg.solve(A, rhs)
        nxt = it.copy(order="F")
        for (i, j), r in idx.items():
            nxt[i, j] = sol[r]
        delta = max(abs(nxt[i, j] - it[i, j]) for (i, j) in idx)
        it = nxt
        if delta < stop_tol:
            break
    return it


def dense_axial_half_step(case, source, T_half, tau, stop_tol, max_sweeps=200):
    """oracles.hpp:117-176: capacity and source frozen at T_half,
    conductivities at the running iterate."""
    grid, mats, cfg = case.grid(), case.materials, case.solver
    idx = _cells(grid)
    it = T_half.copy(order="F")
    for _ in range(max_sweeps):
        A = np.zeros((len(idx), len(idx)))
        rhs = np.zeros(len(idx))
        for i in range(grid.nr()):
            m = grid.col_extent(i)
            mat = mats[grid.layer(i)]
            for j in range(m):
                row = idx[(i, j)]
                eta = grid.control_z(j)
                K = mat.rho() * mat.eval(Property.HeatCapacity, T_half[i, j], cfg.range_policy) / (0.5 * tau)
                A[row, row] += K
                rhs[row] += K * T_half[i, j]
                if j > 0:
                    c = face_lambda(mat, mat, it[i, j - 1], it[i, j], cfg) / (grid.gap_z(j) * eta)
                    A[row, row] += c
                    A[row, idx[(i, j - 1)]] -= c
                if j < m - 1:
                    c = face_lambda(mat, mat, it[i, j], it[i, j + 1], cfg) / (grid.gap_z(j + 1) * eta)
                    A[row, row] += c
                    A[row, idx[(i, j + 1)]] -= c
                elif grid.layer(i) == 0 and not cfg.all_neumann:
                    c = mat.eval(Property.Conductivity, cfg.T0, cfg.range_policy) / (0.5 * grid.width_z(j) * eta)
                    A[row, row] += c
                    rhs[row] += c * cfg.T0
                rhs[row] += apply_lambda_r(grid, mats, T_half, i, j, cfg)
                rhs[row] += joule_power(case, source, i if grid.layer(i) == case.domain.source_layer
                                        else None, T_half[i, j])
        sol = np.linalg.solve(A, rhs)
        nxt = it.copy(order="F")
        for (i, j), r in idx.items():
            nxt[i, j] = sol[r]
        delta = max(abs(nxt[i, j] - it[i, j]) for (i, j) in idx)
        it = nxt
        if delta < stop_tol:
            break
    return it


class Manufactured:
    """The acceptance suite's manufactured solution (acceptance_main.cpp:239-260)."""
    R = Z = 1.0
    rho, cv, lam = 1.0, 1.0, 0.5
    T0, A, gamma = 4.2, 10.0, 5.0

    def amp(self, t):
        return self.A * math.exp(-self.gamma * t)

    def phi(self, r):
        return np.cos(math.pi * r * r / (self.R * self.R))

    def lr_phi(self, r):
        a = math.pi / (self.R * self.R)
        return -4.0 * a * np.sin(a * r * r) - 4.0 * a * a * r * r * np.cos(a * r * r)

    def psi(self, z):
        return np.cos(0.5 * math.pi * z / self.Z)

    def psi_zz(self, z):
        b = 0.5 * math.pi / self.Z
        return -b * b * self.psi(z)

    def exact(self, r, z, t):
        return self.T0 + self.amp(t) * self.phi(r) * self.psi(z)

    def source(self, r, z, t):
        return (self.rho * self.cv * (-self.gamma) * self.amp(t) * self.phi(r) * self.psi(z) -
                self.lam * self.amp(t) * (self.lr_phi(r) * self.psi(z) + self.phi(r) * self.psi_zz(z)))
