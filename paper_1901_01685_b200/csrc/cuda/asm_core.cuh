// asm_core.cuh -- the arithmetic of the GPU assembler (F2), one function per
// phase of an element.  Every expression is written in the operand order of the host element loop
// (csrc/host/discretization.cpp assemble_operator / assemble_mixed_mass) so that, without
// multiply-add contraction (-fmad=false), the element matrices and the gathered CSR values equal
// the host's bit for bit.  The functions are __host__ __device__: assemble.cu runs them as CUDA
// kernels; tests/cpp/asm_emulate.cpp runs the same code serially on the CPU to check the index
// logic and the canonical accumulation order where no GPU is present (test infrastructure only).
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define PMG_HD __host__ __device__ __forceinline__
#else
#define PMG_HD inline
#endif

namespace pmgasm {

constexpr int kMaxP = 5, kMaxN1 = kMaxP + 1, kMaxQ = kMaxN1 * kMaxN1;

struct Tab {  // pmg_asm_table1d with device pointers
    int p;
    const double* B;
    const double* dB;
    const int32_t* first;
};
struct Geo {
    Tab gx, gy;
    int gnx;
    const double *cx, *cy, *w;
};
struct Params {
    int kind, nel, nq, strip;
    int n1, n2;        // p_row + 1, p_col + 1
    const double* wq;  // nel*nq
    Tab row, col;
    Geo geo;
    int dirichlet;     // edge mask of the current patch
    double D[4], v[2], R, pen;
};

// per-element scratch (shared memory on the GPU)
struct Scratch {
    double K[4 * kMaxQ], C[2 * kMaxQ], Mr[kMaxQ];  // Mr doubles as the mass weight W
    double S[4 * kMaxN1 * kMaxQ];                  // stage-1 sums
    double phi[4 * kMaxN1 * kMaxQ], flux[4 * kMaxN1 * kMaxQ], wb[4 * kMaxN1];  // Nitsche traces per (edge, a)
    int bad;
};

// rational map and Jacobian at abscissae (ptx, pty): NurbsPatch::map
PMG_HD void geo_map(const Geo& g, int ptx, int pty, double X[2], double J[2][2]) {
    const int px = g.gx.p, py = g.gy.p;
    const double *Nx = g.gx.B + ptx * (px + 1), *dNx = g.gx.dB + ptx * (px + 1);
    const double *Ny = g.gy.B + pty * (py + 1), *dNy = g.gy.dB + pty * (py + 1);
    const int fx = g.gx.first[ptx], fy = g.gy.first[pty];
    double W = 0, Wx = 0, Wy = 0, S[2] = {0, 0}, Sx[2] = {0, 0}, Sy[2] = {0, 0};
    for (int b = 0; b <= py; ++b)
        for (int a = 0; a <= px; ++a) {
            const int k = (fx + a) + (fy + b) * g.gnx;
            const double wk = g.w[k];
            const double v = Nx[a] * Ny[b] * wk, vx = dNx[a] * Ny[b] * wk, vy = Nx[a] * dNy[b] * wk;
            W += v; Wx += vx; Wy += vy;
            S[0] += v * g.cx[k]; S[1] += v * g.cy[k];
            Sx[0] += vx * g.cx[k]; Sx[1] += vx * g.cy[k];
            Sy[0] += vy * g.cx[k]; Sy[1] += vy * g.cy[k];
        }
    for (int r = 0; r < 2; ++r) {
        X[r] = S[r] / W;
        J[r][0] = (Sx[r] - X[r] * Wx) / W;
        J[r][1] = (Sy[r] - X[r] * Wy) / W;
    }
}

PMG_HD void inv2(const double J[2][2], double G[2][2], double& det) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    G[0][0] = J[1][1] / det;  G[0][1] = -J[0][1] / det;
    G[1][0] = -J[1][0] / det; G[1][1] = J[0][0] / det;
}

// ---- operator: geometric factors at Gauss point q = a + b*nq of element (ex, ey)
PMG_HD void op_point(const Params& P, int ex, int ey, int q, Scratch& s) {
    const int nq = P.nq, a = q % nq, b = q / nq, nqq = nq * nq;
    double X[2], J[2][2], G[2][2], det;
    geo_map(P.geo, ex * nq + a, ey * nq + b, X, J);
    inv2(J, G, det);
    if (!(det > 0)) s.bad = 1;
    const double w = P.wq[ex * nq + a] * P.wq[ey * nq + b] * det;
    for (int r = 0; r < 2; ++r)
        for (int t = 0; t < 2; ++t) {
            double acc = 0;
            for (int m = 0; m < 2; ++m)
                for (int l = 0; l < 2; ++l) acc += G[r][m] * P.D[m * 2 + l] * G[t][l];
            s.K[(r * 2 + t) * nqq + q] = w * acc;
        }
    for (int r = 0; r < 2; ++r) s.C[r * nqq + q] = w * (G[r][0] * P.v[0] + G[r][1] * P.v[1]);
    s.Mr[q] = w * P.R;
}

// ---- operator stage 1: item = (b, i1, i2), sums over the xi points a
PMG_HD void op_stage1(const Params& P, int ex, int item, Scratch& s) {
    const int nq = P.nq, n1 = P.n1, nqq = nq * nq;
    const int i2 = item % n1, i1 = (item / n1) % n1, b = item / (n1 * n1);
    double syy = 0, syd = 0, sdy = 0, sdd = 0;
    for (int a = 0; a < nq; ++a) {
        const int q = a + b * nq;
        const double *Bx = P.row.B + (ex * nq + a) * n1, *dBx = P.row.dB + (ex * nq + a) * n1;
        const double k00 = s.K[q], k01 = s.K[nqq + q], k10 = s.K[2 * nqq + q], k11 = s.K[3 * nqq + q];
        const double c0 = s.C[q], c1 = s.C[nqq + q], m = s.Mr[q];
        syy += k00 * dBx[i1] * dBx[i2] + c0 * Bx[i1] * dBx[i2] + m * Bx[i1] * Bx[i2];
        syd += k01 * dBx[i1] * Bx[i2] + c1 * Bx[i1] * Bx[i2];
        sdy += k10 * Bx[i1] * dBx[i2];
        sdd += k11 * Bx[i1] * Bx[i2];
    }
    const int o = i1 * n1 + i2, nn = n1 * n1;
    s.S[(0 * nq + b) * nn + o] = syy;
    s.S[(1 * nq + b) * nn + o] = syd;
    s.S[(2 * nq + b) * nn + o] = sdy;
    s.S[(3 * nq + b) * nn + o] = sdd;
}

PMG_HD bool edge_on(const Params& P, int edge, int ex, int ey) {
    const bool on = (edge == 0 && ey == 0) || (edge == 1 && ex == P.nel - 1) || (edge == 2 && ey == P.nel - 1) ||
                    (edge == 3 && ex == 0);
    return on && ((P.dirichlet >> edge) & 1);
}

// ---- operator: Nitsche traces of boundary point slot = edge*nq + a (only for edges that are on)
PMG_HD void op_trace(const Params& P, int ex, int ey, int slot, Scratch& s) {
    const int nq = P.nq, n1 = P.n1, nn = n1 * n1, nel = P.nel;
    const int edge = slot / nq, a = slot % nq;
    const bool horiz = (edge == 0 || edge == 2);
    const int e_along = horiz ? ex : ey;
    const int pt_s = e_along * nq + a;
    const int pt_x = horiz ? pt_s : (edge == 1 ? nel * nq + 1 : nel * nq);
    const int pt_y = horiz ? (edge == 2 ? nel * nq + 1 : nel * nq) : pt_s;
    const double ws = P.wq[pt_s];
    double X[2], J[2][2], G[2][2], det;
    geo_map(P.geo, pt_x, pt_y, X, J);
    inv2(J, G, det);
    const double t0 = horiz ? J[0][0] : J[0][1], t1 = horiz ? J[1][0] : J[1][1];
    const double tl = sqrt(t0 * t0 + t1 * t1);
    double nv0, nv1;
    if (edge == 0 || edge == 1) { nv0 = t1 / tl; nv1 = -t0 / tl; }
    else { nv0 = -t1 / tl; nv1 = t0 / tl; }
    const double *Nx = P.row.B + pt_x * n1, *dNx = P.row.dB + pt_x * n1;
    const double *Ny = P.row.B + pt_y * n1, *dNy = P.row.dB + pt_y * n1;
    double* phi = s.phi + slot * nn;
    double* flux = s.flux + slot * nn;
    for (int j = 0; j < n1; ++j)
        for (int i = 0; i < n1; ++i) {
            const double g0 = dNx[i] * Ny[j], g1 = Nx[i] * dNy[j];
            const double gx0 = G[0][0] * g0 + G[1][0] * g1, gx1 = G[0][1] * g0 + G[1][1] * g1;
            const double dg0 = P.D[0] * gx0 + P.D[1] * gx1, dg1 = P.D[2] * gx0 + P.D[3] * gx1;
            phi[i + j * n1] = Nx[i] * Ny[j];
            flux[i + j * n1] = dg0 * nv0 + dg1 * nv1;
        }
    s.wb[slot] = ws * tl;
}

// ---- operator: element-matrix entry te = i1 + j1*n1 (test), tr = i2 + j2*n1 (trial)
PMG_HD double op_entry(const Params& P, int ex, int ey, int te, int tr, const Scratch& s) {
    const int nq = P.nq, n1 = P.n1, nn = n1 * n1;
    const int i1 = te % n1, j1 = te / n1, i2 = tr % n1, j2 = tr / n1;
    const int o = i1 * n1 + i2;
    double e = 0.0;
    for (int b = 0; b < nq; ++b) {
        const double *By = P.row.B + (ey * nq + b) * n1, *dBy = P.row.dB + (ey * nq + b) * n1;
        const double yy = By[j1] * By[j2], yd = By[j1] * dBy[j2], dy = dBy[j1] * By[j2], dd = dBy[j1] * dBy[j2];
        e += yy * s.S[(0 * nq + b) * nn + o] + yd * s.S[(1 * nq + b) * nn + o] + dy * s.S[(2 * nq + b) * nn + o] +
             dd * s.S[(3 * nq + b) * nn + o];
    }
    for (int edge = 0; edge < 4; ++edge) {
        if (!edge_on(P, edge, ex, ey)) continue;
        for (int a = 0; a < nq; ++a) {
            const int slot = edge * nq + a;
            const double* phi = s.phi + slot * nn;
            const double* flux = s.flux + slot * nn;
            e += s.wb[slot] * (-flux[tr] * phi[te] - flux[te] * phi[tr] + P.pen * phi[te] * phi[tr]);
        }
    }
    return e;
}

// ---- mixed mass: weight at Gauss point q
PMG_HD void mass_point(const Params& P, int ex, int ey, int q, Scratch& s) {
    const int nq = P.nq, a = q % nq, b = q / nq;
    double X[2], J[2][2];
    geo_map(P.geo, ex * nq + a, ey * nq + b, X, J);
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    if (!(det > 0)) s.bad = 1;
    s.Mr[q] = P.wq[ex * nq + a] * P.wq[ey * nq + b] * det;
}

// stage 1: item = (b, i1, i2)
PMG_HD void mass_stage1(const Params& P, int ex, int item, Scratch& s) {
    const int nq = P.nq, n1 = P.n1, n2 = P.n2;
    const int i2 = item % n2, i1 = (item / n2) % n1, b = item / (n1 * n2);
    double acc = 0;
    for (int a = 0; a < nq; ++a) {
        const double* Bx = P.row.B + (ex * nq + a) * n1;
        const double* Cx = P.col.B + (ex * nq + a) * n2;
        acc += s.Mr[a + b * nq] * Bx[i1] * Cx[i2];
    }
    s.S[(b * n1 + i1) * n2 + i2] = acc;
}

// entry te = i1 + j1*n1 (row space), tr = i2 + j2*n2 (column space)
PMG_HD double mass_entry(const Params& P, int ey, int te, int tr, const Scratch& s) {
    const int nq = P.nq, n1 = P.n1, n2 = P.n2;
    const int i1 = te % n1, j1 = te / n1, i2 = tr % n2, j2 = tr / n2;
    double e = 0.0;
    for (int b = 0; b < nq; ++b) {
        const double* By = P.row.B + (ey * nq + b) * n1;
        const double* Cy = P.col.B + (ey * nq + b) * n2;
        const double yy = By[j1] * Cy[j2];
        e += yy * s.S[(b * n1 + i1) * n2 + i2];
    }
    return e;
}

// ---- gather: add to `acc` the contributions of one patch to the CSR entry whose row is the local
// DOF (ix, iy) and whose column is the local DOF (jx, jy), in the canonical order
// (include/pmg_asm.h).  E holds the element matrices of element rows e0.. (row-major over ex).
PMG_HD bool gather_entry(const Params& P, const double* E, int e0, int ix, int iy, int jx, int jy, double& acc) {
    const int pr = P.n1 - 1, pc = P.n2 - 1, nel = P.nel;
    const int64_t esz = int64_t(P.n1) * P.n1 * P.n2 * P.n2;
    const int ncl = P.n2 * P.n2;
    int exlo = ix - pr > jx - pc ? ix - pr : jx - pc, exhi = ix < jx ? ix : jx;
    int eylo = iy - pr > jy - pc ? iy - pr : jy - pc, eyhi = iy < jy ? iy : jy;
    if (exlo < 0) exlo = 0;
    if (eylo < 0) eylo = 0;
    if (exhi > nel - 1) exhi = nel - 1;
    if (eyhi > nel - 1) eyhi = nel - 1;
    if (exlo > exhi || eylo > eyhi) return false;
    for (int colour = 0; colour < 2; ++colour)
        for (int ey = eylo; ey <= eyhi; ++ey) {
            if (((ey / P.strip) & 1) != colour) continue;
            for (int ex = exlo; ex <= exhi; ++ex)
                acc += E[(int64_t(ey - e0) * nel + ex) * esz + ((ix - ex) + (iy - ey) * P.n1) * ncl + (jx - ex) +
                         (jy - ey) * P.n2];
        }
    return true;
}

// ---- lump_mass: row sum in ascending column order (host `lump`)
PMG_HD double row_sum(const double* val, int64_t kb, int64_t ke) {
    double s = 0.0;
    for (int64_t k = kb; k < ke; ++k) s += val[k];
    return s;
}

}  // namespace pmgasm
