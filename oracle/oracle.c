/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the three
 * resampling layers of the gradient-Halide "Custom Neural Network Layers"
 * section and their reverse-mode adjoints (VJPs).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, helper or constant with the CUDA product path
 * (paper_1904_12228_b200/csrc/); the product never loads it.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (no FMA contraction,
 * so every coordinate below is the plain left-to-right fp64 evaluation).
 *
 * What the paper fixes and what it does not
 *   The layer formulas are NOT printed in PAPER.md: the listings and the code
 *   comparison figure are dangling \input{}s.  The
 *   definitions follow the standard conventions of the cited layers, as read
 *   in SURVEY.md §8(c) and listed in DESIGN.md "Readings":
 *     STN    — Jaderberg et al., as exposed by PyTorch affine_grid+grid_sample
 *              (the comparison the paper makes).
 *     warp   — FlowNet 2.0 backward warp, out(x) = in(x + flow(x)), pixels
 *              (PAPER.md:30-34).
 *     bslice — HDRNet slice-and-apply: trilinear tent lookup
 *              into an affine-coefficient grid, per-pixel 3x4 affine apply.
 *   Every adjoint is the reverse-mode derivative df(x, dy) of PAPER.md:2239-2241
 *   ("a buffer representing the adjoints"), written as the naive
 *   SCATTER that reverses the forward gather (the form before
 *   any scatter-to-gather conversion).
 *
 * Layouts (all row-major / C-contiguous, fp64):
 *   x     N x C x H x W          theta N x 2 x 3        y  N x C x Ho x Wo
 *   flow  N x 2 x H x W (ch0 = horizontal displacement, pixels)
 *   grid  N x 12 x D x Gh x Gw   (q = 4*o + i, row-major 3x4, bias last)
 *   guide N x H x W
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py
 * (library routines, closed forms, adjoint identity, central FD, brute-force
 * operator matrix, hand-computed golden fixtures).  None is "parity unpinned".
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* threads                                                              */
/* ------------------------------------------------------------------ */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* STN: affine_grid + bilinear grid_sample            */
/* ------------------------------------------------------------------ */

/* Normalised output coordinate of output index j along an axis of length L.
 * align_corners=1: -1 + 2j/(L-1);  align_corners=0: (2j+1)/L - 1. */
static double stn_norm(int j, int L, int ac) {
    if (ac) return -1.0 + (2.0 * (double)j) / (double)(L - 1);
    return (2.0 * (double)j + 1.0) / (double)L - 1.0;
}

/* Un-normalise a grid coordinate g in [-1,1] to pixel units for size L.
 * align_corners=1: (g+1)(L-1)/2;  align_corners=0: ((g+1)L - 1)/2. */
static double stn_unnorm(double g, int L, int ac) {
    if (ac) return (g + 1.0) * (double)(L - 1) / 2.0;
    return ((g + 1.0) * (double)L - 1.0) / 2.0;
}

/* d(pixel coordinate)/d(grid coordinate). */
static double stn_unnorm_scale(int L, int ac) {
    return ac ? (double)(L - 1) / 2.0 : (double)L / 2.0;
}

/* Border padding: clamp the coordinate to [0, L-1]; the clamp's derivative
 * is 1 strictly inside and 0 otherwise (PyTorch's convention, R3). */
static double clamp_coord(double v, int L, double *dclamp) {
    if (v <= 0.0) { *dclamp = 0.0; return 0.0; }
    if (v >= (double)(L - 1)) { *dclamp = 0.0; return (double)(L - 1); }
    *dclamp = 1.0;
    return v;
}

/* Value of plane p (H x W) at integer tap (yy, xx), zero outside. */
static double tap(const double *p, int H, int W, long yy, long xx) {
    if (yy < 0 || yy >= H || xx < 0 || xx >= W) return 0.0;
    return p[yy * (long)W + xx];
}

/* Sample coordinate of STN output pixel (n, i, j) in input pixel units. */
static void stn_coord(const double *th, int H, int W, int Ho, int Wo, int ac,
                      int i, int j, double *xt, double *yt, double *ix, double *iy) {
    *xt = stn_norm(j, Wo, ac);
    *yt = stn_norm(i, Ho, ac);
    double gx = th[0] * (*xt) + th[1] * (*yt) + th[2];
    double gy = th[3] * (*xt) + th[4] * (*yt) + th[5];
    *ix = stn_unnorm(gx, W, ac);
    *iy = stn_unnorm(gy, H, ac);
}

/* Bilinear sample of plane p at (ix, iy): floor cell (x0,y0), fractions. */
static double bilinear(const double *p, int H, int W, double ix, double iy) {
    double x0 = floor(ix), y0 = floor(iy);
    double fx = ix - x0, fy = iy - y0;
    long X0 = (long)x0, Y0 = (long)y0;
    double v00 = tap(p, H, W, Y0, X0), v01 = tap(p, H, W, Y0, X0 + 1);
    double v10 = tap(p, H, W, Y0 + 1, X0), v11 = tap(p, H, W, Y0 + 1, X0 + 1);
    return (1.0 - fy) * ((1.0 - fx) * v00 + fx * v01) + fy * ((1.0 - fx) * v10 + fx * v11);
}

/* Y[n,c,i,j] = bilinear(X[n,c], ix(i,j), iy(i,j)). */
void oracle_stn_fwd(const double *x, const double *theta, int N, int C, int H, int W,
                    int Ho, int Wo, int ac, int border, double *y) {
    long nrow = (long)N * Ho;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < nrow; r++) {
        int n = (int)(r / Ho), i = (int)(r % Ho);
        const double *th = theta + 6L * n;
        for (int j = 0; j < Wo; j++) {
            double xt, yt, ix, iy, d;
            stn_coord(th, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
            if (border) { ix = clamp_coord(ix, W, &d); iy = clamp_coord(iy, H, &d); }
            for (int c = 0; c < C; c++) {
                const double *p = x + ((long)n * C + c) * H * (long)W;
                y[(((long)n * C + c) * Ho + i) * (long)Wo + j] = bilinear(p, H, W, ix, iy);
            }
        }
    }
}

/* Reverse mode of oracle_stn_fwd.
 *   dx     : naive scatter of dy*w onto the four taps.
 *   dtheta : d_ix = sum_c dy*[(1-fy)(V01-V00)+fy(V11-V10)], d_iy likewise,
 *            d_g = d_i * unnormalise-scale * clamp-derivative,
 *            dtheta[0,:] += d_gx*[xt,yt,1], dtheta[1,:] += d_gy*[xt,yt,1].
 * Either output may be NULL. */
void oracle_stn_bwd(const double *x, const double *theta, const double *dy, int N, int C,
                    int H, int W, int Ho, int Wo, int ac, int border, double *dx,
                    double *dtheta) {
    if (dx) {
        long planes = (long)N * C;
#pragma omp parallel for schedule(static)
        for (long pc = 0; pc < planes; pc++) {
            int n = (int)(pc / C);
            const double *th = theta + 6L * n;
            double *dp = dx + pc * H * (long)W;
            const double *g = dy + pc * Ho * (long)Wo;
            memset(dp, 0, sizeof(double) * (size_t)H * W);
            for (int i = 0; i < Ho; i++)
                for (int j = 0; j < Wo; j++) {
                    double xt, yt, ix, iy, d;
                    stn_coord(th, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                    if (border) { ix = clamp_coord(ix, W, &d); iy = clamp_coord(iy, H, &d); }
                    double x0 = floor(ix), y0 = floor(iy);
                    double fx = ix - x0, fy = iy - y0;
                    long X0 = (long)x0, Y0 = (long)y0;
                    double gv = g[(long)i * Wo + j];
                    double w[4] = {(1.0 - fy) * (1.0 - fx), (1.0 - fy) * fx,
                                   fy * (1.0 - fx), fy * fx};
                    long ty[4] = {Y0, Y0, Y0 + 1, Y0 + 1}, tx[4] = {X0, X0 + 1, X0, X0 + 1};
                    for (int t = 0; t < 4; t++)
                        if (ty[t] >= 0 && ty[t] < H && tx[t] >= 0 && tx[t] < W)
                            dp[ty[t] * W + tx[t]] += w[t] * gv;
                }
        }
    }
    if (dtheta) {
#pragma omp parallel for schedule(static)
        for (int n = 0; n < N; n++) {
            const double *th = theta + 6L * n;
            double acc[6] = {0, 0, 0, 0, 0, 0};
            double sx = stn_unnorm_scale(W, ac), sy = stn_unnorm_scale(H, ac);
            for (int i = 0; i < Ho; i++)
                for (int j = 0; j < Wo; j++) {
                    double xt, yt, ix, iy, cgx = 1.0, cgy = 1.0;
                    stn_coord(th, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                    if (border) { ix = clamp_coord(ix, W, &cgx); iy = clamp_coord(iy, H, &cgy); }
                    double x0 = floor(ix), y0 = floor(iy);
                    double fx = ix - x0, fy = iy - y0;
                    long X0 = (long)x0, Y0 = (long)y0;
                    double dix = 0.0, diy = 0.0;
                    for (int c = 0; c < C; c++) {
                        const double *p = x + ((long)n * C + c) * H * (long)W;
                        double gv = dy[(((long)n * C + c) * Ho + i) * (long)Wo + j];
                        double v00 = tap(p, H, W, Y0, X0), v01 = tap(p, H, W, Y0, X0 + 1);
                        double v10 = tap(p, H, W, Y0 + 1, X0), v11 = tap(p, H, W, Y0 + 1, X0 + 1);
                        dix += gv * ((1.0 - fy) * (v01 - v00) + fy * (v11 - v10));
                        diy += gv * ((1.0 - fx) * (v10 - v00) + fx * (v11 - v01));
                    }
                    double dgx = dix * sx * cgx, dgy = diy * sy * cgy;
                    acc[0] += dgx * xt; acc[1] += dgx * yt; acc[2] += dgx;
                    acc[3] += dgy * xt; acc[4] += dgy * yt; acc[5] += dgy;
                }
            for (int k = 0; k < 6; k++) dtheta[6L * n + k] = acc[k];
        }
    }
}

/* ------------------------------------------------------------------ */
/* Warp: FlowNet 2.0 per-pixel warp                   */
/* ------------------------------------------------------------------ */

/* Y[n,c,y,x] = bilinear(X[n,c], x + flow[n,0,y,x], y + flow[n,1,y,x]). */
void oracle_warp_fwd(const double *x, const double *flow, int N, int C, int H, int W,
                     int border, double *y) {
    long nrow = (long)N * H;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < nrow; r++) {
        int n = (int)(r / H), yy = (int)(r % H);
        const double *fu = flow + (2L * n) * H * (long)W, *fv = fu + (long)H * W;
        for (int xx = 0; xx < W; xx++) {
            double d;
            double ix = (double)xx + fu[(long)yy * W + xx];
            double iy = (double)yy + fv[(long)yy * W + xx];
            if (border) { ix = clamp_coord(ix, W, &d); iy = clamp_coord(iy, H, &d); }
            for (int c = 0; c < C; c++) {
                const double *p = x + ((long)n * C + c) * H * (long)W;
                y[(((long)n * C + c) * H + yy) * (long)W + xx] = bilinear(p, H, W, ix, iy);
            }
        }
    }
}

/* Reverse mode of oracle_warp_fwd: dx by naive scatter, dflow = (d_ix, d_iy)
 * times the clamp derivative (no normalisation scale: flow is in pixels). */
void oracle_warp_bwd(const double *x, const double *flow, const double *dy, int N, int C,
                     int H, int W, int border, double *dx, double *dflow) {
    if (dx) {
        long planes = (long)N * C;
#pragma omp parallel for schedule(static)
        for (long pc = 0; pc < planes; pc++) {
            int n = (int)(pc / C);
            const double *fu = flow + (2L * n) * H * (long)W, *fv = fu + (long)H * W;
            double *dp = dx + pc * H * (long)W;
            const double *g = dy + pc * H * (long)W;
            memset(dp, 0, sizeof(double) * (size_t)H * W);
            for (int yy = 0; yy < H; yy++)
                for (int xx = 0; xx < W; xx++) {
                    double d;
                    double ix = (double)xx + fu[(long)yy * W + xx];
                    double iy = (double)yy + fv[(long)yy * W + xx];
                    if (border) { ix = clamp_coord(ix, W, &d); iy = clamp_coord(iy, H, &d); }
                    double x0 = floor(ix), y0 = floor(iy);
                    double fx = ix - x0, fy = iy - y0;
                    long X0 = (long)x0, Y0 = (long)y0;
                    double gv = g[(long)yy * W + xx];
                    double w[4] = {(1.0 - fy) * (1.0 - fx), (1.0 - fy) * fx,
                                   fy * (1.0 - fx), fy * fx};
                    long ty[4] = {Y0, Y0, Y0 + 1, Y0 + 1}, tx[4] = {X0, X0 + 1, X0, X0 + 1};
                    for (int t = 0; t < 4; t++)
                        if (ty[t] >= 0 && ty[t] < H && tx[t] >= 0 && tx[t] < W)
                            dp[ty[t] * W + tx[t]] += w[t] * gv;
                }
        }
    }
    if (dflow) {
        long nrow = (long)N * H;
#pragma omp parallel for schedule(static)
        for (long r = 0; r < nrow; r++) {
            int n = (int)(r / H), yy = (int)(r % H);
            const double *fu = flow + (2L * n) * H * (long)W, *fv = fu + (long)H * W;
            for (int xx = 0; xx < W; xx++) {
                double cgx = 1.0, cgy = 1.0;
                double ix = (double)xx + fu[(long)yy * W + xx];
                double iy = (double)yy + fv[(long)yy * W + xx];
                if (border) { ix = clamp_coord(ix, W, &cgx); iy = clamp_coord(iy, H, &cgy); }
                double x0 = floor(ix), y0 = floor(iy);
                double fx = ix - x0, fy = iy - y0;
                long X0 = (long)x0, Y0 = (long)y0;
                double dix = 0.0, diy = 0.0;
                for (int c = 0; c < C; c++) {
                    const double *p = x + ((long)n * C + c) * H * (long)W;
                    double gv = dy[(((long)n * C + c) * H + yy) * (long)W + xx];
                    double v00 = tap(p, H, W, Y0, X0), v01 = tap(p, H, W, Y0, X0 + 1);
                    double v10 = tap(p, H, W, Y0 + 1, X0), v11 = tap(p, H, W, Y0 + 1, X0 + 1);
                    dix += gv * ((1.0 - fy) * (v01 - v00) + fy * (v11 - v10));
                    diy += gv * ((1.0 - fx) * (v10 - v00) + fx * (v11 - v01));
                }
                dflow[((2L * n) * H + yy) * (long)W + xx] = dix * cgx;
                dflow[((2L * n + 1) * H + yy) * (long)W + xx] = diy * cgy;
            }
        }
    }
}

/* ------------------------------------------------------------------ */
/* Bilateral slice-apply: HDRNet                       */
/* ------------------------------------------------------------------ */

static long clampi(long v, long lo, long hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* Cell-centre coordinates of pixel (yy, xx) with guide value gd:
 *   cx = (x+1/2) Gw/W - 1/2,  cy = (y+1/2) Gh/H - 1/2,  cz = gd*D - 1/2. */
static void bs_coord(int yy, int xx, double gd, int H, int W, int D, int Gh, int Gw,
                     double *cx, double *cy, double *cz) {
    *cx = ((double)xx + 0.5) * (double)Gw / (double)W - 0.5;
    *cy = ((double)yy + 0.5) * (double)Gh / (double)H - 0.5;
    *cz = gd * (double)D - 0.5;
}

/* A_q = sum over the 8 taps of wx*wy*wz*grid[n,q,clamp z,clamp y,clamp x];
 * taps floor(c), floor(c)+1 per axis with weights 1-frac, frac; the index is
 * clamped to the grid while the weight uses the unclamped position. */
static void bs_slice(const double *gr, int D, int Gh, int Gw, double cx, double cy,
                     double cz, double A[12]) {
    double x0 = floor(cx), y0 = floor(cy), z0 = floor(cz);
    double fx = cx - x0, fy = cy - y0, fz = cz - z0;
    for (int q = 0; q < 12; q++) A[q] = 0.0;
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2; b++)
            for (int e = 0; e < 2; e++) {
                double w = (e ? fz : 1.0 - fz) * (b ? fy : 1.0 - fy) * (a ? fx : 1.0 - fx);
                long zi = clampi((long)z0 + e, 0, D - 1), yi = clampi((long)y0 + b, 0, Gh - 1),
                     xi = clampi((long)x0 + a, 0, Gw - 1);
                for (int q = 0; q < 12; q++)
                    A[q] += w * gr[(((long)q * D + zi) * Gh + yi) * Gw + xi];
            }
}

/* Y_o = sum_{i<3} A_{4o+i} X_i + A_{4o+3}. */
void oracle_bslice_fwd(const double *grid, const double *guide, const double *x, int N, int H,
                       int W, int D, int Gh, int Gw, double *y) {
    long nrow = (long)N * H;
#pragma omp parallel for schedule(static)
    for (long r = 0; r < nrow; r++) {
        int n = (int)(r / H), yy = (int)(r % H);
        const double *gr = grid + (long)n * 12 * D * Gh * Gw;
        long HW = (long)H * W;
        for (int xx = 0; xx < W; xx++) {
            long pix = (long)yy * W + xx;
            double cx, cy, cz, A[12];
            bs_coord(yy, xx, guide[(long)n * HW + pix], H, W, D, Gh, Gw, &cx, &cy, &cz);
            bs_slice(gr, D, Gh, Gw, cx, cy, cz, A);
            double xi[4] = {x[(3L * n + 0) * HW + pix], x[(3L * n + 1) * HW + pix],
                            x[(3L * n + 2) * HW + pix], 1.0};
            for (int o = 0; o < 3; o++) {
                double s = 0.0;
                for (int i = 0; i < 4; i++) s += A[4 * o + i] * xi[i];
                y[(3L * n + o) * HW + pix] = s;
            }
        }
    }
}

/* Reverse mode of oracle_bslice_fwd.
 *   dx_i    = sum_o dy_o A_{4o+i}
 *   dguide  = D * sum_o dy_o sum_i Xt_i (A_hi - A_lo)_{4o+i}, A_lo/A_hi the
 *             spatial bilinear slices at planes clamp(z0), clamp(z0+1)
 *             (dA/dcz = A_hi - A_lo; zero when both planes clamp together)
 *   dgrid   : naive scatter of wx*wy*wz*dy_o*Xt_i onto the 8 taps.
 * Any output may be NULL. */
void oracle_bslice_bwd(const double *grid, const double *guide, const double *x,
                       const double *dy, int N, int H, int W, int D, int Gh, int Gw,
                       double *dgrid, double *dguide, double *dx) {
    long HW = (long)H * W;
    long GS = 12L * D * Gh * Gw;
    if (dx || dguide) {
        long nrow = (long)N * H;
#pragma omp parallel for schedule(static)
        for (long r = 0; r < nrow; r++) {
            int n = (int)(r / H), yy = (int)(r % H);
            const double *gr = grid + (long)n * GS;
            for (int xx = 0; xx < W; xx++) {
                long pix = (long)yy * W + xx;
                double cx, cy, cz, A[12];
                bs_coord(yy, xx, guide[(long)n * HW + pix], H, W, D, Gh, Gw, &cx, &cy, &cz);
                bs_slice(gr, D, Gh, Gw, cx, cy, cz, A);
                double g[3] = {dy[(3L * n + 0) * HW + pix], dy[(3L * n + 1) * HW + pix],
                               dy[(3L * n + 2) * HW + pix]};
                if (dx)
                    for (int i = 0; i < 3; i++) {
                        double s = 0.0;
                        for (int o = 0; o < 3; o++) s += g[o] * A[4 * o + i];
                        dx[(3L * n + i) * HW + pix] = s;
                    }
                if (dguide) {
                    /* spatial slices at the two (clamped) z planes */
                    double z0 = floor(cz);
                    double Alo[12], Ahi[12];
                    double x0 = floor(cx), y0 = floor(cy);
                    double fx = cx - x0, fy = cy - y0;
                    long zl = clampi((long)z0, 0, D - 1), zh = clampi((long)z0 + 1, 0, D - 1);
                    for (int q = 0; q < 12; q++) { Alo[q] = 0.0; Ahi[q] = 0.0; }
                    for (int a = 0; a < 2; a++)
                        for (int b = 0; b < 2; b++) {
                            double w = (b ? fy : 1.0 - fy) * (a ? fx : 1.0 - fx);
                            long yi = clampi((long)y0 + b, 0, Gh - 1),
                                 xi = clampi((long)x0 + a, 0, Gw - 1);
                            for (int q = 0; q < 12; q++) {
                                Alo[q] += w * gr[(((long)q * D + zl) * Gh + yi) * Gw + xi];
                                Ahi[q] += w * gr[(((long)q * D + zh) * Gh + yi) * Gw + xi];
                            }
                        }
                    double xt[4] = {x[(3L * n + 0) * HW + pix], x[(3L * n + 1) * HW + pix],
                                    x[(3L * n + 2) * HW + pix], 1.0};
                    double s = 0.0;
                    for (int o = 0; o < 3; o++)
                        for (int i = 0; i < 4; i++)
                            s += g[o] * xt[i] * (Ahi[4 * o + i] - Alo[4 * o + i]);
                    dguide[(long)n * HW + pix] = (double)D * s;
                }
            }
        }
    }
    if (dgrid) {
#pragma omp parallel for schedule(static)
        for (int n = 0; n < N; n++) {
            const double *gd = guide + (long)n * HW;
            double *dg = dgrid + (long)n * GS;
            memset(dg, 0, sizeof(double) * (size_t)GS);
            for (int yy = 0; yy < H; yy++)
                for (int xx = 0; xx < W; xx++) {
                    long pix = (long)yy * W + xx;
                    double cx, cy, cz;
                    bs_coord(yy, xx, gd[pix], H, W, D, Gh, Gw, &cx, &cy, &cz);
                    double x0 = floor(cx), y0 = floor(cy), z0 = floor(cz);
                    double fx = cx - x0, fy = cy - y0, fz = cz - z0;
                    double xt[4] = {x[(3L * n + 0) * HW + pix], x[(3L * n + 1) * HW + pix],
                                    x[(3L * n + 2) * HW + pix], 1.0};
                    double g[3] = {dy[(3L * n + 0) * HW + pix], dy[(3L * n + 1) * HW + pix],
                                   dy[(3L * n + 2) * HW + pix]};
                    for (int a = 0; a < 2; a++)
                        for (int b = 0; b < 2; b++)
                            for (int e = 0; e < 2; e++) {
                                double w = (e ? fz : 1.0 - fz) * (b ? fy : 1.0 - fy) *
                                           (a ? fx : 1.0 - fx);
                                long zi = clampi((long)z0 + e, 0, D - 1),
                                     yi = clampi((long)y0 + b, 0, Gh - 1),
                                     xi = clampi((long)x0 + a, 0, Gw - 1);
                                for (int o = 0; o < 3; o++)
                                    for (int i = 0; i < 4; i++)
                                        dg[(((long)(4 * o + i) * D + zi) * Gh + yi) * Gw + xi] +=
                                            w * g[o] * xt[i];
                            }
                }
        }
    }
}

/* ------------------------------------------------------------------ */
/* 2-D convolution layer        */
/* ------------------------------------------------------------------ */
/* The paper's gather ("output(x) = input(x - r.x) *
 * kernel(r.x)") extended to 2-D and channels, centred so the output has the
 * input's size (reading R10):
 *   y[n,co,y,x] = sum_{ci<Ci, ry<kh, rx<kw} x[n,ci, y-ry+ph, x-rx+pw] * k[co,ci,ry,rx]
 * with ph = kh/2, pw = kw/2 (integer division) and zero outside [0,H)x[0,W).
 * x: N x Ci x H x W, k: Co x Ci x kh x kw, y: N x Co x H x W.                */
static double conv_in(const double *xc, int H, int W, long u, long v) {
    return (u >= 0 && u < H && v >= 0 && v < W) ? xc[u * W + v] : 0.0;
}

void oracle_conv_fwd(const double *x, const double *k, int N, int Ci, int Co, int H, int W,
                     int kh, int kw, double *y) {
    const long HW = (long)H * W;
    const int ph = kh / 2, pw = kw / 2;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int co = 0; co < Co; co++)
            for (int yy = 0; yy < H; yy++)
                for (int xx = 0; xx < W; xx++) {
                    double s = 0.0;
                    for (int ci = 0; ci < Ci; ci++)
                        for (int ry = 0; ry < kh; ry++)
                            for (int rx = 0; rx < kw; rx++)
                                s += conv_in(x + ((long)n * Ci + ci) * HW, H, W, yy - ry + ph, xx - rx + pw) *
                                     k[(((long)co * Ci + ci) * kh + ry) * kw + rx];
                    y[((long)n * Co + co) * HW + (long)yy * W + xx] = s;
                }
}

/* Adjoints (VJP) of the layer above.
 *   dx: the NAIVE SCATTER of PAPER.md:709-713, "d_input(ro.y - ro.x) +=
 *       d_output(ro.y) * kernel(ro.x)": every output element adds g*k into the
 *       input elements it read (the form before scatter-to-gather conversion).
 *       Race-free: OpenMP over samples, each writes only its own dx slice.
 *   dk: the plain definition dk[co,ci,ry,rx] = sum_{n,y,x} dy[n,co,y,x] *
 *       x[n,ci,y-ry+ph,x-rx+pw] (the layer is bilinear in x and k).           */
void oracle_conv_bwd(const double *x, const double *k, const double *dy, int N, int Ci, int Co,
                     int H, int W, int kh, int kw, double *dx, double *dk) {
    const long HW = (long)H * W;
    const int ph = kh / 2, pw = kw / 2;
    if (dx) {
#pragma omp parallel for schedule(static)
        for (int n = 0; n < N; n++) {
            double *dxn = dx + (long)n * Ci * HW;
            memset(dxn, 0, sizeof(double) * (size_t)(Ci * HW));
            for (int co = 0; co < Co; co++)
                for (int yy = 0; yy < H; yy++)
                    for (int xx = 0; xx < W; xx++) {
                        const double g = dy[((long)n * Co + co) * HW + (long)yy * W + xx];
                        for (int ci = 0; ci < Ci; ci++)
                            for (int ry = 0; ry < kh; ry++)
                                for (int rx = 0; rx < kw; rx++) {
                                    const long u = yy - ry + ph, v = xx - rx + pw;
                                    if (u >= 0 && u < H && v >= 0 && v < W)
                                        dxn[(long)ci * HW + u * W + v] +=
                                            g * k[(((long)co * Ci + ci) * kh + ry) * kw + rx];
                                }
                    }
        }
    }
    if (dk) {
#pragma omp parallel for collapse(2) schedule(static)
        for (int co = 0; co < Co; co++)
            for (int ci = 0; ci < Ci; ci++)
                for (int ry = 0; ry < kh; ry++)
                    for (int rx = 0; rx < kw; rx++) {
                        double s = 0.0;
                        for (int n = 0; n < N; n++)
                            for (int yy = 0; yy < H; yy++)
                                for (int xx = 0; xx < W; xx++)
                                    s += dy[((long)n * Co + co) * HW + (long)yy * W + xx] *
                                         conv_in(x + ((long)n * Ci + ci) * HW, H, W, yy - ry + ph, xx - rx + pw);
                        dk[(((long)co * Ci + ci) * kh + ry) * kw + rx] = s;
                    }
    }
}

/* ------------------------------------------------------------------ */
/* Checkpointing study          */
/* ------------------------------------------------------------------ */
/* convolved = in (*) kernel, loss = sum (convolved - target)^2,
 * d_in = "a cross correlation of 2*(convolved-target) with kernel".
 * Single channel, the layer of oracle_conv_fwd with Ci = Co = 1 (zero padding,
 * centred; R11).  Written as its definition: the residual
 * r = 2 (conv(in) - target), then the naive-scatter adjoint of the convolution.
 * in, target, d_in: N x H x W; k: kh x kw.                                    */
void oracle_convloss_grad(const double *in, const double *k, const double *target, int N, int H,
                          int W, int kh, int kw, double *d_in) {
    const long HW = (long)H * W;
    double *r = (double *)malloc(sizeof(double) * (size_t)(N * HW));
    oracle_conv_fwd(in, k, N, 1, 1, H, W, kh, kw, r);
    for (long i = 0; i < N * HW; i++) r[i] = 2.0 * (r[i] - target[i]);
    oracle_conv_bwd(in, k, r, N, 1, 1, H, W, kh, kw, d_in, NULL);
    free(r);
}

/* Upsampling by 4: output(x, y) = input(x/4, y/4), integer
 * division; x: N x C x H x W, y: N x C x 4H x 4W.  Adjoint as the naive scatter
 * d_input(x/4, y/4) += d_output(x, y).                                        */
void oracle_upsample4_fwd(const double *x, int N, int C, int H, int W, double *y) {
    const long Wo = 4L * W, Ho = 4L * H;
    for (long nc = 0; nc < (long)N * C; nc++)
        for (long yy = 0; yy < Ho; yy++)
            for (long xx = 0; xx < Wo; xx++)
                y[(nc * Ho + yy) * Wo + xx] = x[(nc * H + yy / 4) * W + xx / 4];
}

void oracle_upsample4_bwd(const double *dy, int N, int C, int H, int W, double *dx) {
    const long Wo = 4L * W, Ho = 4L * H;
    memset(dx, 0, sizeof(double) * (size_t)N * C * H * W);
    for (long nc = 0; nc < (long)N * C; nc++)
        for (long yy = 0; yy < Ho; yy++)
            for (long xx = 0; xx < Wo; xx++)
                dx[(nc * H + yy / 4) * W + xx / 4] += dy[(nc * Ho + yy) * Wo + xx];
}

/* ------------------------------------------------------------------ */
/* STN variants ("changing the        */
/* interpolation scheme ... or interpolating over more dimensions")    */
/* ------------------------------------------------------------------ */
/* Bicubic: Keys' cubic convolution with A = -0.75 over the 4 x 4 taps
 * floor(i) - 1 .. floor(i) + 2 per axis, zeros outside (the convention of
 * PyTorch grid_sample(mode='bicubic'), R12).  Coordinates as R1.   */
static const double CUBIC_A = -0.75;
static double cubic1(double x) { return ((CUBIC_A + 2.0) * x - (CUBIC_A + 3.0)) * x * x + 1.0; }
static double cubic2(double x) { return ((CUBIC_A * x - 5.0 * CUBIC_A) * x + 8.0 * CUBIC_A) * x - 4.0 * CUBIC_A; }
static double dcubic1(double x) { return (3.0 * (CUBIC_A + 2.0) * x - 2.0 * (CUBIC_A + 3.0)) * x; }
static double dcubic2(double x) { return (3.0 * CUBIC_A * x - 10.0 * CUBIC_A) * x + 8.0 * CUBIC_A; }
static void cubic_w(double t, double w[4], double dw[4]) {
    w[0] = cubic2(t + 1.0); w[1] = cubic1(t); w[2] = cubic1(1.0 - t); w[3] = cubic2(2.0 - t);
    dw[0] = dcubic2(t + 1.0); dw[1] = dcubic1(t); dw[2] = -dcubic1(1.0 - t); dw[3] = -dcubic2(2.0 - t);
}

void oracle_stn_bicubic_fwd(const double *x, const double *theta, int N, int C, int H, int W,
                            int Ho, int Wo, int ac, double *y) {
    const long HW = (long)H * W, P = (long)Ho * Wo;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int i = 0; i < Ho; i++)
                for (int j = 0; j < Wo; j++) {
                    double xt, yt, ix, iy, wx[4], wy[4], d[4];
                    stn_coord(theta + 6L * n, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                    const double x0 = floor(ix), y0 = floor(iy);
                    cubic_w(ix - x0, wx, d);
                    cubic_w(iy - y0, wy, d);
                    const double *p = x + ((long)n * C + c) * HW;
                    double s = 0.0;
                    for (int a = 0; a < 4; a++)
                        for (int b = 0; b < 4; b++)
                            s += wy[a] * wx[b] * tap(p, H, W, (long)y0 - 1 + a, (long)x0 - 1 + b);
                    y[((long)n * C + c) * P + (long)i * Wo + j] = s;
                }
}

/* Adjoint: d_input by the naive scatter of every tap, d_theta by the chain rule
 * through d(weights)/dt and the un-normalisation scale, summed over pixels. */
void oracle_stn_bicubic_bwd(const double *x, const double *theta, const double *dy, int N, int C,
                            int H, int W, int Ho, int Wo, int ac, double *dx, double *dtheta) {
    const long HW = (long)H * W, P = (long)Ho * Wo;
    const double sx = stn_unnorm_scale(W, ac), sy = stn_unnorm_scale(H, ac);
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; n++) {
        if (dx) memset(dx + (long)n * C * HW, 0, sizeof(double) * (size_t)(C * HW));
        double dth[6] = {0, 0, 0, 0, 0, 0};
        for (int i = 0; i < Ho; i++)
            for (int j = 0; j < Wo; j++) {
                double xt, yt, ix, iy, wx[4], wy[4], dwx[4], dwy[4];
                stn_coord(theta + 6L * n, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                const double x0 = floor(ix), y0 = floor(iy);
                cubic_w(ix - x0, wx, dwx);
                cubic_w(iy - y0, wy, dwy);
                double gix = 0.0, giy = 0.0;
                for (int c = 0; c < C; c++) {
                    const double g = dy[((long)n * C + c) * P + (long)i * Wo + j];
                    const double *p = x + ((long)n * C + c) * HW;
                    for (int a = 0; a < 4; a++)
                        for (int b = 0; b < 4; b++) {
                            const long yy = (long)y0 - 1 + a, xx = (long)x0 - 1 + b;
                            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                            const double v = p[yy * W + xx];
                            if (dx) dx[((long)n * C + c) * HW + yy * W + xx] += g * wy[a] * wx[b];
                            gix += g * wy[a] * dwx[b] * v;
                            giy += g * dwy[a] * wx[b] * v;
                        }
                }
                const double gx = gix * sx, gy = giy * sy;
                dth[0] += gx * xt; dth[1] += gx * yt; dth[2] += gx;
                dth[3] += gy * xt; dth[4] += gy * yt; dth[5] += gy;
            }
        if (dtheta)
            for (int k = 0; k < 6; k++) dtheta[6L * n + k] = dth[k];
    }
}

/* Volumetric STN: theta N x 3 x 4, x N x C x D x H x W, output N x C x Do x Ho x Wo;
 * normalised (x_t, y_t, z_t) per R1 on each axis, (g_x, g_y, g_z) = theta [x_t, y_t, z_t, 1],
 * trilinear tent over the 8 taps, zeros outside (PyTorch 5-D affine_grid + grid_sample). */
static double tap3(const double *p, int D, int H, int W, long zz, long yy, long xx) {
    if (zz < 0 || zz >= D || yy < 0 || yy >= H || xx < 0 || xx >= W) return 0.0;
    return p[(zz * H + yy) * (long)W + xx];
}

static void stn3_coord(const double *th, int D, int H, int W, int Do, int Ho, int Wo, int ac, int k,
                       int i, int j, double t[3], double pix[3]) {
    t[0] = stn_norm(j, Wo, ac);
    t[1] = stn_norm(i, Ho, ac);
    t[2] = stn_norm(k, Do, ac);
    const int L[3] = {W, H, D};
    for (int r = 0; r < 3; r++) {
        const double g = th[4 * r] * t[0] + th[4 * r + 1] * t[1] + th[4 * r + 2] * t[2] + th[4 * r + 3];
        pix[r] = stn_unnorm(g, L[r], ac);
    }
}

void oracle_stn3d_fwd(const double *x, const double *theta, int N, int C, int D, int H, int W, int Do,
                      int Ho, int Wo, int ac, double *y) {
    const long V = (long)D * H * W, Po = (long)Do * Ho * Wo;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int k = 0; k < Do; k++)
                for (int i = 0; i < Ho; i++)
                    for (int j = 0; j < Wo; j++) {
                        double t[3], q[3];
                        stn3_coord(theta + 12L * n, D, H, W, Do, Ho, Wo, ac, k, i, j, t, q);
                        const double x0 = floor(q[0]), y0 = floor(q[1]), z0 = floor(q[2]);
                        const double f[3] = {q[0] - x0, q[1] - y0, q[2] - z0};
                        const double *p = x + ((long)n * C + c) * V;
                        double s = 0.0;
                        for (int e = 0; e < 8; e++) {
                            const int a = e & 1, b = (e >> 1) & 1, d = e >> 2;
                            const double w = (a ? f[0] : 1.0 - f[0]) * (b ? f[1] : 1.0 - f[1]) * (d ? f[2] : 1.0 - f[2]);
                            s += w * tap3(p, D, H, W, (long)z0 + d, (long)y0 + b, (long)x0 + a);
                        }
                        y[((long)n * C + c) * Po + ((long)k * Ho + i) * Wo + j] = s;
                    }
}

void oracle_stn3d_bwd(const double *x, const double *theta, const double *dy, int N, int C, int D, int H,
                      int W, int Do, int Ho, int Wo, int ac, double *dx, double *dtheta) {
    const long V = (long)D * H * W, Po = (long)Do * Ho * Wo;
    const double sc[3] = {stn_unnorm_scale(W, ac), stn_unnorm_scale(H, ac), stn_unnorm_scale(D, ac)};
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; n++) {
        if (dx) memset(dx + (long)n * C * V, 0, sizeof(double) * (size_t)(C * V));
        double dth[12] = {0};
        for (int k = 0; k < Do; k++)
            for (int i = 0; i < Ho; i++)
                for (int j = 0; j < Wo; j++) {
                    double t[3], q[3];
                    stn3_coord(theta + 12L * n, D, H, W, Do, Ho, Wo, ac, k, i, j, t, q);
                    const double x0 = floor(q[0]), y0 = floor(q[1]), z0 = floor(q[2]);
                    const double f[3] = {q[0] - x0, q[1] - y0, q[2] - z0};
                    double gq[3] = {0, 0, 0};
                    for (int c = 0; c < C; c++) {
                        const double g = dy[((long)n * C + c) * Po + ((long)k * Ho + i) * Wo + j];
                        const double *p = x + ((long)n * C + c) * V;
                        for (int e = 0; e < 8; e++) {
                            const int a = e & 1, b = (e >> 1) & 1, d = e >> 2;
                            const double wx = a ? f[0] : 1.0 - f[0], wy = b ? f[1] : 1.0 - f[1],
                                         wz = d ? f[2] : 1.0 - f[2];
                            const long zz = (long)z0 + d, yy = (long)y0 + b, xx = (long)x0 + a;
                            if (zz < 0 || zz >= D || yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                            const double v = p[(zz * H + yy) * W + xx];
                            if (dx) dx[((long)n * C + c) * V + (zz * H + yy) * W + xx] += g * wx * wy * wz;
                            gq[0] += g * (a ? 1.0 : -1.0) * wy * wz * v;
                            gq[1] += g * wx * (b ? 1.0 : -1.0) * wz * v;
                            gq[2] += g * wx * wy * (d ? 1.0 : -1.0) * v;
                        }
                    }
                    for (int r = 0; r < 3; r++) {
                        const double gg = gq[r] * sc[r];
                        dth[4 * r] += gg * t[0]; dth[4 * r + 1] += gg * t[1];
                        dth[4 * r + 2] += gg * t[2]; dth[4 * r + 3] += gg;
                    }
                }
        if (dtheta)
            for (int r = 0; r < 12; r++) dtheta[12L * n + r] = dth[r];
    }
}

/* ------------------------------------------------------------------ */
/* Diagnostics: kink-straddling sample coordinates       */
/* ------------------------------------------------------------------ */
/* Number of sample coordinates (each axis counted separately) within tol px of an
 * integer, where the floor cell -- and so the one-sided derivative (R8) --
 * is decided by the last bits of the coordinate.  Reported next to parity results. */
static int near_int(double v, double tol) { return fabs(v - floor(v + 0.5)) <= tol; }

long oracle_stn_kinks(const double *theta, int N, int H, int W, int Ho, int Wo, int ac, double tol) {
    long cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
    for (int n = 0; n < N; n++)
        for (int i = 0; i < Ho; i++)
            for (int j = 0; j < Wo; j++) {
                double xt, yt, ix, iy;
                stn_coord(theta + 6L * n, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                cnt += near_int(ix, tol) + near_int(iy, tol);
            }
    return cnt;
}

long oracle_warp_kinks(const double *flow, int N, int H, int W, double tol) {
    const long HW = (long)H * W;
    long cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
    for (int n = 0; n < N; n++)
        for (long p = 0; p < HW; p++) {
            const double ix = (double)(p % W) + flow[(2L * n) * HW + p];
            const double iy = (double)(p / W) + flow[(2L * n + 1) * HW + p];
            cnt += near_int(ix, tol) + near_int(iy, tol);
        }
    return cnt;
}

/* bilateral slice: the guide axis c_z = guide * D - 1/2 (the spatial cell coordinates
 * are fixed by the shapes) */
long oracle_bslice_kinks(const double *guide, int N, int H, int W, int D, double tol) {
    const long T = (long)N * H * W;
    long cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
    for (long p = 0; p < T; p++) cnt += near_int(guide[p] * (double)D - 0.5, tol);
    return cnt;
}

/* Lanczos-3 STN ("changing the interpolation scheme", PAPER.md:28;
 * DESIGN.md R13): 6 x 6 taps floor(i)-2 .. floor(i)+3 per axis with the (unnormalised)
 * Lanczos kernel L(x) = sinc(x) sinc(x/3) for |x| < 3, sinc(x) = sin(pi x)/(pi x),
 * zeros outside the image; coordinates as R1.                                  */
static const double PI_ = 3.14159265358979323846;
static double lanczos3(double x) {
    if (x == 0.0) return 1.0;
    if (fabs(x) >= 3.0) return 0.0;
    const double px = PI_ * x;
    return 3.0 * sin(px) * sin(px / 3.0) / (px * px);
}
static double dlanczos3(double x) {
    if (x == 0.0 || fabs(x) >= 3.0) return 0.0;
    const double px = PI_ * x, s1 = sin(px), s3 = sin(px / 3.0), c1 = cos(px), c3 = cos(px / 3.0);
    return 3.0 * (PI_ * c1 * s3 + (PI_ / 3.0) * s1 * c3) / (px * px) - 6.0 * s1 * s3 / (px * px * x);
}
static void lanczos_w(double t, double w[6], double dw[6]) {
    for (int m = 0; m < 6; m++) { w[m] = lanczos3(t + 2.0 - m); dw[m] = dlanczos3(t + 2.0 - m); }
}

void oracle_stn_lanczos_fwd(const double *x, const double *theta, int N, int C, int H, int W,
                            int Ho, int Wo, int ac, double *y) {
    const long HW = (long)H * W, P = (long)Ho * Wo;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < N; n++)
        for (int c = 0; c < C; c++)
            for (int i = 0; i < Ho; i++)
                for (int j = 0; j < Wo; j++) {
                    double xt, yt, ix, iy, wx[6], wy[6], d[6];
                    stn_coord(theta + 6L * n, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                    const double x0 = floor(ix), y0 = floor(iy);
                    lanczos_w(ix - x0, wx, d);
                    lanczos_w(iy - y0, wy, d);
                    const double *p = x + ((long)n * C + c) * HW;
                    double s = 0.0;
                    for (int a = 0; a < 6; a++)
                        for (int b = 0; b < 6; b++)
                            s += wy[a] * wx[b] * tap(p, H, W, (long)y0 - 2 + a, (long)x0 - 2 + b);
                    y[((long)n * C + c) * P + (long)i * Wo + j] = s;
                }
}

void oracle_stn_lanczos_bwd(const double *x, const double *theta, const double *dy, int N, int C,
                            int H, int W, int Ho, int Wo, int ac, double *dx, double *dtheta) {
    const long HW = (long)H * W, P = (long)Ho * Wo;
    const double sx = stn_unnorm_scale(W, ac), sy = stn_unnorm_scale(H, ac);
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N; n++) {
        if (dx) memset(dx + (long)n * C * HW, 0, sizeof(double) * (size_t)(C * HW));
        double dth[6] = {0, 0, 0, 0, 0, 0};
        for (int i = 0; i < Ho; i++)
            for (int j = 0; j < Wo; j++) {
                double xt, yt, ix, iy, wx[6], wy[6], dwx[6], dwy[6];
                stn_coord(theta + 6L * n, H, W, Ho, Wo, ac, i, j, &xt, &yt, &ix, &iy);
                const double x0 = floor(ix), y0 = floor(iy);
                lanczos_w(ix - x0, wx, dwx);
                lanczos_w(iy - y0, wy, dwy);
                double gix = 0.0, giy = 0.0;
                for (int c = 0; c < C; c++) {
                    const double g = dy[((long)n * C + c) * P + (long)i * Wo + j];
                    const double *p = x + ((long)n * C + c) * HW;
                    for (int a = 0; a < 6; a++)
                        for (int b = 0; b < 6; b++) {
                            const long yy = (long)y0 - 2 + a, xx = (long)x0 - 2 + b;
                            if (yy < 0 || yy >= H || xx < 0 || xx >= W) continue;
                            const double v = p[yy * W + xx];
                            if (dx) dx[((long)n * C + c) * HW + yy * W + xx] += g * wy[a] * wx[b];
                            gix += g * wy[a] * dwx[b] * v;
                            giy += g * dwy[a] * wx[b] * v;
                        }
                }
                const double gx = gix * sx, gy = giy * sy;
                dth[0] += gx * xt; dth[1] += gx * yt; dth[2] += gx;
                dth[3] += gy * xt; dth[4] += gy * yt; dth[5] += gy;
            }
        if (dtheta)
            for (int k = 0; k < 6; k++) dtheta[6L * n + k] = dth[k];
    }
}

double oracle_lanczos3(double x) { return lanczos3(x); }
double oracle_dlanczos3(double x) { return dlanczos3(x); }
