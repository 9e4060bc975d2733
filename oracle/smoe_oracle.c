/*
 * oracle/smoe_oracle.c -- CPU ORACLE FOR THE R-SMoE HOT PATH.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2510_05814_b200/) never imports, links or calls it,
 * and this file shares no code, header, constant or helper with it.
 *
 * Plain, slow, single-threaded, fp64.  Every pixel is evaluated against EVERY
 * kernel (dense), with the paper's truncation rule applied per pair.  There is
 * no tiling, no binning, no reordering: the rasterised method reaches exactly
 * this truncated model, so the dense definition is the oracle.
 *
 * Citations: P:n = PAPER.md line n (arxiv 2510.05814), S:n = SPEC.md line n.
 *
 *   steered kernel      K_j(x) = exp(-1/2 (x-mu_j)^T Sigma_j^-1 (x-mu_j))  Eq.(3)
 *   soft gate           w_j = pi_j K_j / sum_i pi_i K_i                    Eq.(4)
 *   regression          y(x) = sum_j m_j(x) w_j(x)                          Eq.(2)
 *   block subset        sum restricted to kernels affecting the block      Eq.(5)
 *   truncation          99% confidence ellipse, out-of-ellipse discarded
 *   Cholesky            Sigma = L L^T, L = [[l11,0],[l21,l22]]
 *   experts             constant m_j or linear m_j + W_j (x-mu_j)   (north_star)
 *   bounding box        square, side = major axis of the 99% ellipse
 *   loss                MSE over H*W*C (reading Q8)
 *   PSNR                10 log10(1/MSE) on [0,1]-clamped images
 *
 * Readings of the paper: R^2 = chi2_2(0.99) = 2 ln 100
 * for both the cull and the box (Q1); the cull is applied in forward and
 * backward (Q2); gates are normalised over the same truncated set (Q3); a
 * pixel with no contributing kernel renders 0 (Q7); pixel (row i, col j) is
 * centred at (j, i); SR samples y at x_src = (j+1/2) W/out_W - 1/2 (Q16).
 *
 * Parameter layout (caller arrays, fp64 here):
 *   mu[K][2] = (mu_x, mu_y); chol[K][3] = (l11, l21, l22); log_pi[K] = ln pi;
 *   expert[K][C][E], E = 1 + 2*order: (m_c) or (m_c, Wx_c, Wy_c).
 * Gradient layout grad[K][Pk], Pk = 6 + C*E:
 *   (mu_x, mu_y, l11, l21, l22, log_pi, expert block in the expert layout).
 *
 * Gradients here are derived through Sigma^-1 (matrix calculus,
 * d(d^2)/dSigma = -q q^T with q = Sigma^-1 delta, then dSigma/dL), a route
 * independent of the whitened form used on the GPU; both are pinned to
 * central finite differences (tests/test_oracle.py).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* chi-square quantile with 2 dof at 0.99: the chi2_2 CDF is 1 - exp(-x/2),
 * so x = -2 ln(1 - 0.99) ("99% confidence interval"). */
double oracle_R2_99(void) { return -2.0 * log(1.0 - 0.99); }

/* Sigma = L L^T: s11 = l11^2, s12 = l11 l21, s22 = l21^2 + l22^2 */
void oracle_cov(const double *chol, double *s11, double *s12, double *s22)
{
    double l11 = chol[0], l21 = chol[1], l22 = chol[2];
    *s11 = l11 * l11;
    *s12 = l11 * l21;
    *s22 = l21 * l21 + l22 * l22;
}

/* Mahalanobis distance (x-mu)^T Sigma^-1 (x-mu) with the explicit 2x2
 * inverse (adjugate / determinant); the exponent of Eq. (3). */
double oracle_d2(const double *mu, const double *chol, double px, double py)
{
    double s11, s12, s22;
    oracle_cov(chol, &s11, &s12, &s22);
    double det = s11 * s22 - s12 * s12;
    double dx = px - mu[0], dy = py - mu[1];
    return (s22 * dx * dx - 2.0 * s12 * dx * dy + s11 * dy * dy) / det;
}

/* Largest eigenvalue of Sigma, closed form for a symmetric 2x2 matrix
 * ("major and minor axes derived from the kernel's covariance"). */
double oracle_lambda_max(const double *chol)
{
    double s11, s12, s22;
    oracle_cov(chol, &s11, &s12, &s22);
    double h = 0.5 * (s11 - s22);
    return 0.5 * (s11 + s22) + sqrt(h * h + s12 * s12);
}

/* Square bounding box of the truncation ellipse: half side
 * r = sqrt(R2 * lambda_max) (so the full side is the major axis 2r).
 * A pixel (output grid out_H x out_W) is inside the box iff its source-space
 * sample point lies in [mu - r, mu + r] per axis (reading Q5 / rule T).
 * Output column j samples x_src = (j + 1/2) W / out_W - 1/2, so the box
 * covers j in [ceil((mu-r+1/2) out_W/W - 1/2), floor((mu+r+1/2) out_W/W - 1/2)].
 * pixbox[k] = (x_lo, x_hi, y_lo, y_hi) clipped to the image; tilebox[k] =
 * (tx0, tx1, ty0, ty1) with 16x16 blocks; all -1 when empty. */
void oracle_boxes(int K, const double *mu, const double *chol, double R2,
                  int H, int W, int out_H, int out_W,
                  int *pixbox, int *tilebox, double *half_side)
{
    double sx = (double)out_W / (double)W, sy = (double)out_H / (double)H;
    for (int k = 0; k < K; k++) {
        double r = sqrt(R2 * oracle_lambda_max(chol + 3 * k));
        if (half_side) half_side[k] = r;
        double mx = mu[2 * k], my = mu[2 * k + 1];
        double xl = ceil((mx - r + 0.5) * sx - 0.5);
        double xh = floor((mx + r + 0.5) * sx - 0.5);
        double yl = ceil((my - r + 0.5) * sy - 0.5);
        double yh = floor((my + r + 0.5) * sy - 0.5);
        if (xl < 0) xl = 0;
        if (yl < 0) yl = 0;
        if (xh > out_W - 1) xh = out_W - 1;
        if (yh > out_H - 1) yh = out_H - 1;
        int *pb = pixbox + 4 * k, *tb = tilebox + 4 * k;
        if (!(xl <= xh && yl <= yh)) {
            pb[0] = pb[1] = pb[2] = pb[3] = -1;
            tb[0] = tb[1] = tb[2] = tb[3] = -1;
            continue;
        }
        pb[0] = (int)xl; pb[1] = (int)xh; pb[2] = (int)yl; pb[3] = (int)yh;
        tb[0] = pb[0] / 16; tb[1] = pb[1] / 16; tb[2] = pb[2] / 16; tb[3] = pb[3] / 16;
    }
}

/* Box modes (reading Q4): 0 = square box of half side
 * R sqrt(lambda_max(Sigma)) (the default); 1 = axis-aligned
 * box of the ellipse, half sides R sqrt(Sigma_xx) = R l11 and
 * R sqrt(Sigma_yy) = R sqrt(l21^2 + l22^2); 2 = exact: the blocks of the
 * mode-1 box whose rectangle of pixel-centre sample points meets the
 * ellipse d^2 <= R2.  Every mode lists every block holding a pixel inside
 * the ellipse, so pixels do not depend on the mode; only the lists do. */
static void half_sides(const double *chol, double R2, int mode, double *rx, double *ry)
{
    if (mode == 0) {
        double r = sqrt(R2 * oracle_lambda_max(chol));
        *rx = r;
        *ry = r;
    } else {
        double s11, s12, s22;
        oracle_cov(chol, &s11, &s12, &s22);
        *rx = sqrt(R2 * s11);
        *ry = sqrt(R2 * s22);
    }
}

/* min of d^2 = delta^T Sigma^-1 delta over the rectangle [x0,x1] x [y0,y1]
 * (source coordinates): 0 if mu is inside, else the least of the four edge
 * minima (each a 1-D quadratic minimised over a segment). */
double oracle_rect_min_d2(const double *mu, const double *chol, double x0, double x1, double y0, double y1)
{
    if (mu[0] >= x0 && mu[0] <= x1 && mu[1] >= y0 && mu[1] <= y1) return 0.0;
    double s11, s12, s22;
    oracle_cov(chol, &s11, &s12, &s22);
    double det = s11 * s22 - s12 * s12;
    double p = s22 / det, q = -s12 / det, r = s11 / det;   /* Sigma^-1 = [[p, q], [q, r]] */
    double best = 1e300;
    double xs[2] = {x0, x1}, ys[2] = {y0, y1};
    for (int e = 0; e < 2; e++) {
        /* edge x = xs[e]: minimise over dy in [y0 - mu_y, y1 - mu_y] */
        double dx = xs[e] - mu[0];
        double dy = -q * dx / r;
        if (dy < y0 - mu[1]) dy = y0 - mu[1];
        if (dy > y1 - mu[1]) dy = y1 - mu[1];
        double v = p * dx * dx + 2.0 * q * dx * dy + r * dy * dy;
        if (v < best) best = v;
        /* edge y = ys[e] */
        dy = ys[e] - mu[1];
        dx = -q * dy / p;
        if (dx < x0 - mu[0]) dx = x0 - mu[0];
        if (dx > x1 - mu[0]) dx = x1 - mu[0];
        v = p * dx * dx + 2.0 * q * dx * dy + r * dy * dy;
        if (v < best) best = v;
    }
    return best;
}

/* Boxes and (block, kernel) pairs under a box mode on the out_H x out_W
 * raster: tilebox[K][4] (candidate blocks, -1 when empty) and up to `cap`
 * pairs (tiles[i], kers[i]) in kernel-major, row-major block order; returns
 * the number of pairs (all of them counted even beyond cap).  In mode 2 the
 * rectangle of block (tx, ty) spans the source points of its output pixel
 * centres: x in [(16 tx + 1/2) W/out_W - 1/2, (min(16 tx + 15, out_W-1) +
 * 1/2) W/out_W - 1/2], likewise y. */
long long oracle_block_pairs(int K, const double *mu, const double *chol, double R2, int H, int W,
                             int out_H, int out_W, int mode, int *tilebox, int *tiles, int *kers,
                             long long cap)
{
    double sx = (double)out_W / (double)W, sy = (double)out_H / (double)H;
    int nx = (out_W + 15) / 16;
    long long n = 0;
    for (int k = 0; k < K; k++) {
        double rx, ry;
        half_sides(chol + 3 * k, R2, mode, &rx, &ry);
        double mx = mu[2 * k], my = mu[2 * k + 1];
        double xl = ceil((mx - rx + 0.5) * sx - 0.5), xh = floor((mx + rx + 0.5) * sx - 0.5);
        double yl = ceil((my - ry + 0.5) * sy - 0.5), yh = floor((my + ry + 0.5) * sy - 0.5);
        if (xl < 0) xl = 0;
        if (yl < 0) yl = 0;
        if (xh > out_W - 1) xh = out_W - 1;
        if (yh > out_H - 1) yh = out_H - 1;
        int *tb = tilebox + 4 * k;
        if (!(xl <= xh && yl <= yh)) { tb[0] = tb[1] = tb[2] = tb[3] = -1; continue; }
        tb[0] = (int)xl / 16; tb[1] = (int)xh / 16; tb[2] = (int)yl / 16; tb[3] = (int)yh / 16;
        for (int ty = tb[2]; ty <= tb[3]; ty++)
            for (int tx = tb[0]; tx <= tb[1]; tx++) {
                if (mode == 2) {
                    int jx1 = 16 * tx + 15 < out_W - 1 ? 16 * tx + 15 : out_W - 1;
                    int iy1 = 16 * ty + 15 < out_H - 1 ? 16 * ty + 15 : out_H - 1;
                    double x0 = (16 * tx + 0.5) / sx - 0.5, x1 = (jx1 + 0.5) / sx - 0.5;
                    double y0 = (16 * ty + 0.5) / sy - 0.5, y1 = (iy1 + 0.5) / sy - 0.5;
                    if (!(oracle_rect_min_d2(mu + 2 * k, chol + 3 * k, x0, x1, y0, y1) <= R2)) continue;
                }
                if (n < cap) { tiles[n] = ty * nx + tx; kers[n] = k; }
                n++;
            }
    }
    return n;
}

/* Margins of the box-mode decisions (rule P1 for modes 1, 2): per kernel,
 * the smallest distance of its four mode box edges (mapped to the output
 * raster) to an integer and, in mode 2, the smallest |rect_min_d2 - R2|
 * over its candidate blocks (1e300 when none). */
void oracle_mode_margins(int K, const double *mu, const double *chol, double R2, int H, int W,
                         int out_H, int out_W, int mode, double *edge_gap, double *rect_gap)
{
    double sx = (double)out_W / (double)W, sy = (double)out_H / (double)H;
    for (int k = 0; k < K; k++) {
        double rx, ry;
        half_sides(chol + 3 * k, R2, mode, &rx, &ry);
        double mx = mu[2 * k], my = mu[2 * k + 1];
        double e[4] = {(mx - rx + 0.5) * sx - 0.5, (mx + rx + 0.5) * sx - 0.5,
                       (my - ry + 0.5) * sy - 0.5, (my + ry + 0.5) * sy - 0.5};
        double eg = 1.0;
        for (int q = 0; q < 4; q++) {
            double f = fabs(e[q] - floor(e[q] + 0.5));
            if (f < eg) eg = f;
        }
        edge_gap[k] = eg;
        double rg = 1e300;
        if (mode == 2) {
            double xl = ceil(e[0]), xh = floor(e[1]), yl = ceil(e[2]), yh = floor(e[3]);
            if (xl < 0) xl = 0;
            if (yl < 0) yl = 0;
            if (xh > out_W - 1) xh = out_W - 1;
            if (yh > out_H - 1) yh = out_H - 1;
            if (xl <= xh && yl <= yh)
                for (int ty = (int)yl / 16; ty <= (int)yh / 16; ty++)
                    for (int tx = (int)xl / 16; tx <= (int)xh / 16; tx++) {
                        int jx1 = 16 * tx + 15 < out_W - 1 ? 16 * tx + 15 : out_W - 1;
                        int iy1 = 16 * ty + 15 < out_H - 1 ? 16 * ty + 15 : out_H - 1;
                        double v = oracle_rect_min_d2(mu + 2 * k, chol + 3 * k, (16 * tx + 0.5) / sx - 0.5,
                                                      (jx1 + 0.5) / sx - 0.5, (16 * ty + 0.5) / sy - 0.5,
                                                      (iy1 + 0.5) / sy - 0.5);
                        if (fabs(v - R2) < rg) rg = fabs(v - R2);
                    }
        }
        rect_gap[k] = rg;
    }
}

/* Expert value m_jc(x) = m_c (+ Wx_c dx + Wy_c dy for the linear expert). */
static double expert_value(const double *e, int order, double dx, double dy)
{
    if (order == 0) return e[0];
    return e[0] + e[1] * dx + e[2] * dy;
}

/* Gate numerator pi_j K_j(x) under the truncation rule: 0 when the pixel lies
 * outside the 99% ellipse (d^2 > R2), else exp(log_pi) exp(-d^2/2). */
static double gate_num(const double *mu, const double *chol, double log_pi,
                       double px, double py, double R2, double *d2_out)
{
    double d2 = oracle_d2(mu, chol, px, py);
    if (d2_out) *d2_out = d2;
    if (!(d2 <= R2)) return 0.0;
    return exp(log_pi) * exp(-0.5 * d2);
}

/* Gates of Eq. (4) at one point, normalised over the truncated set (Q3). */
void oracle_gates(int K, const double *mu, const double *chol, const double *log_pi,
                  double px, double py, double R2, double *w, double *D_out)
{
    double D = 0.0;
    for (int j = 0; j < K; j++) {
        w[j] = gate_num(mu + 2 * j, chol + 3 * j, log_pi[j], px, py, R2, NULL);
        D += w[j];
    }
    for (int j = 0; j < K; j++) w[j] = D > 0.0 ? w[j] / D : 0.0;
    if (D_out) *D_out = D;
}

/* Regression head: 0 = SMoE, y = sum_j m_j(x) w_j(x) with the soft gates of
 * Eq. (4) (Eq. 2); 1 = RBF / GaussianImage-style weighted sum of
 * kernels y = sum_j m_j(x) pi_j K_j(x) (Eq. 1; pi_j = 1 there, kept
 * as a multiplier here so log_pi = 0 reproduces Eq. 1 exactly). */
static int g_head = 0;
void oracle_set_head(int head) { g_head = head; }

/* y(x) of Eq. (2)/(5) (or Eq. 1) at one source-space point, all C channels. */
static void eval_point(int K, int C, int order, const double *mu, const double *chol,
                       const double *log_pi, const double *expert,
                       double px, double py, double R2, double *y, double *D_out)
{
    int E = 1 + 2 * order;
    double D = 0.0;
    for (int c = 0; c < C; c++) y[c] = 0.0;
    for (int j = 0; j < K; j++) {
        double g = gate_num(mu + 2 * j, chol + 3 * j, log_pi[j], px, py, R2, NULL);
        if (g == 0.0) continue;
        double dx = px - mu[2 * j], dy = py - mu[2 * j + 1];
        D += g;
        for (int c = 0; c < C; c++)
            y[c] += g * expert_value(expert + (size_t)(j * C + c) * E, order, dx, dy);
    }
    if (g_head == 0)
        for (int c = 0; c < C; c++) y[c] = D > 0.0 ? y[c] / D : 0.0;  /* Q7 */
    if (D_out) *D_out = D;
}

/* Render on an out_H x out_W raster (native SR by re-sampling),
 * output rows [row0, row1). y[C][row1-row0][out_W], D[row1-row0][out_W]. */
void oracle_render(int K, int C, int order, const double *mu, const double *chol,
                   const double *log_pi, const double *expert, int H, int W,
                   int out_H, int out_W, int row0, int row1, double R2,
                   double *y, double *D)
{
    int nr = row1 - row0;
    double yc[8];
    for (int i = row0; i < row1; i++) {
        double py = (i + 0.5) * H / out_H - 0.5;
        for (int jx = 0; jx < out_W; jx++) {
            double px = (jx + 0.5) * W / out_W - 0.5;
            double Dp;
            eval_point(K, C, order, mu, chol, log_pi, expert, px, py, R2, yc, &Dp);
            size_t o = (size_t)(i - row0) * out_W + jx;
            for (int c = 0; c < C; c++) y[(size_t)c * nr * out_W + o] = yc[c];
            if (D) D[o] = Dp;
        }
    }
}

/* y(x) at n arbitrary source-space points (sampled parity at full size). */
void oracle_render_points(int K, int C, int order, const double *mu, const double *chol,
                          const double *log_pi, const double *expert, int n,
                          const double *xs, const double *ys, double R2,
                          double *y /*[n][C]*/, double *D /*[n]*/)
{
    for (int p = 0; p < n; p++)
        eval_point(K, C, order, mu, chol, log_pi, expert, xs[p], ys[p], R2,
                   y + (size_t)p * C, D ? D + p : NULL);
}

/* Per-pixel gradient contribution of kernel j at pixel (px,py) given the
 * pixel's y, D and e_c = dL/dy_c.  Adds into g[Pk] and |term| into a[Pk].
 *   s = dL/d(d^2) = -1/2 g G,  G = sum_c e_c (m_jc(x) - y_c) / D
 *   d(d^2)/dmu = -2 q, q = Sigma^-1 delta;  d(d^2)/dSigma_ab = -q_a q_b
 *   Sigma = L L^T gives dSigma/dl11 = [[2 l11, l21],[l21, 0]],
 *   dSigma/dl21 = [[0, l11],[l11, 2 l21]], dSigma/dl22 = [[0,0],[0, 2 l22]]. */
static void add_pair_grad(int C, int order, const double *mu, const double *chol,
                          double log_pi, const double *e_j, double px, double py,
                          const double *yv, double D, const double *ev, const double *eva,
                          double R2, double *g, double *a, double *b)
{
    int E = 1 + 2 * order;
    double d2;
    double gn = gate_num(mu, chol, log_pi, px, py, R2, &d2);
    if (gn == 0.0) return;                       /* culled pair */
    double dx = px - mu[0], dy = py - mu[1];
    double s11, s12, s22;
    oracle_cov(chol, &s11, &s12, &s22);
    double det = s11 * s22 - s12 * s12;
    double q1 = (s22 * dx - s12 * dy) / det, q2 = (-s12 * dx + s11 * dy) / det;
    /* SMoE: dy_c/dg_j = (m_jc(x) - y_c)/D, dy_c/dm_jc(x) = w_j = g_j/D;
     * RBF (Eq. 1): dy_c/dg_j = m_jc(x), dy_c/dm_jc(x) = g_j. */
    double w = g_head == 0 ? gn / D : gn;
    double G = 0.0;
    for (int c = 0; c < C; c++)
        G += ev[c] * (expert_value(e_j + c * E, order, dx, dy) - (g_head == 0 ? yv[c] : 0.0));
    if (g_head == 0) G /= D;
    double s = -0.5 * gn * G;
    /* operand scale of the same term (b): every difference in it -- the
     * residual y - t inside e_c and m_jc(x) - y_c inside G -- replaced by the
     * sum of its operands' magnitudes, the scale of its rounding error in
     * any finite-precision evaluation (forward error of a sum <= u * sum of
     * |operands|).  Test tolerance scale only; not part of the gradient. */
    double Gb = 0.0;
    for (int c = 0; c < C; c++)
        Gb += eva[c] * (fabs(expert_value(e_j + c * E, order, dx, dy)) + (g_head == 0 ? fabs(yv[c]) : 0.0));
    if (g_head == 0) Gb /= D;
    double sb = 0.5 * gn * Gb;
    double l11 = chol[0], l21 = chol[1], l22 = chol[2];
    double t[64];
    int n = 0;
    /* gate path */
    t[n++] = s * (-2.0 * q1);                                   /* mu_x */
    t[n++] = s * (-2.0 * q2);                                   /* mu_y */
    t[n++] = s * -(q1 * q1 * 2.0 * l11 + 2.0 * q1 * q2 * l21);  /* l11 */
    t[n++] = s * -(2.0 * q1 * q2 * l11 + q2 * q2 * 2.0 * l21);  /* l21 */
    t[n++] = s * -(q2 * q2 * 2.0 * l22);                        /* l22 */
    t[n++] = gn * G;                                            /* log_pi: dg/dlog_pi = g */
    /* expert path: dy_c/dm_jc(x) = w */
    for (int c = 0; c < C; c++) {
        double ew = ev[c] * w;
        t[n++] = ew;                                            /* m_c */
        if (order == 1) {
            t[n++] = ew * dx;                                   /* Wx_c */
            t[n++] = ew * dy;                                   /* Wy_c */
            /* dm_jc(x)/dmu = -(Wx_c, Wy_c): accumulated separately below */
        }
    }
    int P = n;
    if (b) {
        /* operand scale: gate-path terms with |s| -> sb, expert-path terms
         * with |e_c| -> eva[c] */
        double tb[6] = {2.0 * fabs(q1), 2.0 * fabs(q2), fabs(q1 * q1 * 2.0 * l11) + fabs(2.0 * q1 * q2 * l21),
                        fabs(2.0 * q1 * q2 * l11) + fabs(q2 * q2 * 2.0 * l21), fabs(q2 * q2 * 2.0 * l22), 2.0};
        for (int i = 0; i < 6; i++) b[i] += sb * tb[i];
        int m = 6;
        for (int c = 0; c < C; c++) {
            double ew = eva[c] * w;
            b[m++] += ew;
            if (order == 1) {
                b[m++] += ew * fabs(dx);
                b[m++] += ew * fabs(dy);
            }
        }
        if (order == 1)
            for (int c = 0; c < C; c++) {
                b[0] += eva[c] * w * fabs(e_j[c * E + 1]);
                b[1] += eva[c] * w * fabs(e_j[c * E + 2]);
            }
    }
    if (order == 1) {
        double emx = 0.0, emy = 0.0;
        for (int c = 0; c < C; c++) {
            emx += ev[c] * w * e_j[c * E + 1];
            emy += ev[c] * w * e_j[c * E + 2];
        }
        t[0] -= emx;
        t[1] -= emy;
        if (a) { a[0] += fabs(emx); a[1] += fabs(emy); }
    }
    for (int i = 0; i < P; i++) {
        g[i] += t[i];
        if (a) a[i] += fabs(t[i]);
    }
}

/* Loss, PSNR partial sums and the exact analytic gradient of
 * L = (1/(H W C)) sum_{x,c} (y_c(x) - t_c(x))^2 over rows [row0,row1).
 * grad/grad_abs: [K][Pk] (overwritten); stats = (SSE, SSE on clamped images,
 * number of uncovered pixels).  target[C][H][W]. */
void oracle_loss_grad(int K, int C, int order, const double *mu, const double *chol,
                      const double *log_pi, const double *expert, int H, int W,
                      const double *target, int row0, int row1, double R2,
                      double *grad, double *grad_abs, double *grad_opnd, double *stats)
{
    int E = 1 + 2 * order, Pk = 6 + C * E;
    memset(grad, 0, sizeof(double) * (size_t)K * Pk);
    if (grad_abs) memset(grad_abs, 0, sizeof(double) * (size_t)K * Pk);
    if (grad_opnd) memset(grad_opnd, 0, sizeof(double) * (size_t)K * Pk);
    double sse = 0.0, ssec = 0.0, unc = 0.0, N = (double)H * W * C;
    double yv[8], ev[8], eva[8];
    for (int i = row0; i < row1; i++) {
        for (int jx = 0; jx < W; jx++) {
            double px = jx, py = i, D;
            eval_point(K, C, order, mu, chol, log_pi, expert, px, py, R2, yv, &D);
            for (int c = 0; c < C; c++) {
                double t = target[(size_t)c * H * W + (size_t)i * W + jx];
                double r = yv[c] - t;
                sse += r * r;
                double yc = yv[c] < 0 ? 0 : (yv[c] > 1 ? 1 : yv[c]);
                double tc = t < 0 ? 0 : (t > 1 ? 1 : t);
                ssec += (yc - tc) * (yc - tc);
                ev[c] = 2.0 * r / N;                 /* dL/dy_c */
                eva[c] = 2.0 * (fabs(yv[c]) + fabs(t)) / N;
            }
            if (!(D > 0.0)) { unc += 1.0; continue; } /* y = 0 is constant: no gradient */
            for (int j = 0; j < K; j++)
                add_pair_grad(C, order, mu + 2 * j, chol + 3 * j, log_pi[j],
                              expert + (size_t)j * C * E, px, py, yv, D, ev, eva, R2,
                              grad + (size_t)j * Pk, grad_abs ? grad_abs + (size_t)j * Pk : NULL,
                              grad_opnd ? grad_opnd + (size_t)j * Pk : NULL);
        }
    }
    stats[0] = sse; stats[1] = ssec; stats[2] = unc;
}

/* Gradient of the full-image loss for a SUBSET of kernels (sampled parity at
 * sizes where the dense all-pixel loop is too slow).  For each selected kernel
 * only pixels inside its box can contribute; y and D at those pixels are still
 * evaluated densely over all K.  grad/grad_abs: [nsel][Pk]. */
void oracle_grad_kernels(int K, int C, int order, const double *mu, const double *chol,
                         const double *log_pi, const double *expert, int H, int W,
                         const double *target, double R2, int nsel, const int *sel,
                         double *grad, double *grad_abs, double *grad_opnd)
{
    int E = 1 + 2 * order, Pk = 6 + C * E;
    double N = (double)H * W * C;
    double yv[8], ev[8], eva[8];
    memset(grad, 0, sizeof(double) * (size_t)nsel * Pk);
    if (grad_abs) memset(grad_abs, 0, sizeof(double) * (size_t)nsel * Pk);
    if (grad_opnd) memset(grad_opnd, 0, sizeof(double) * (size_t)nsel * Pk);
    for (int s = 0; s < nsel; s++) {
        int j = sel[s];
        int pb[4], tb[4];
        oracle_boxes(1, mu + 2 * j, chol + 3 * j, R2, H, W, H, W, pb, tb, NULL);
        if (pb[0] < 0) continue;
        for (int i = pb[2]; i <= pb[3]; i++)
            for (int jx = pb[0]; jx <= pb[1]; jx++) {
                double px = jx, py = i, D;
                if (!(oracle_d2(mu + 2 * j, chol + 3 * j, px, py) <= R2)) continue;
                eval_point(K, C, order, mu, chol, log_pi, expert, px, py, R2, yv, &D);
                for (int c = 0; c < C; c++) {
                    double t = target[(size_t)c * H * W + (size_t)i * W + jx];
                    ev[c] = 2.0 * (yv[c] - t) / N;
                    eva[c] = 2.0 * (fabs(yv[c]) + fabs(t)) / N;
                }
                add_pair_grad(C, order, mu + 2 * j, chol + 3 * j, log_pi[j],
                              expert + (size_t)j * C * E, px, py, yv, D, ev, eva, R2,
                              grad + (size_t)s * Pk, grad_abs ? grad_abs + (size_t)s * Pk : NULL,
                              grad_opnd ? grad_opnd + (size_t)s * Pk : NULL);
            }
    }
}

/* Margin report for parity-input conditioning (SURVEY §8(c) rule P1): for
 * each kernel, the smallest |d^2 - R2| over the output-grid sample points in
 * a one-pixel-padded box, and the smallest distance of the four box-edge
 * coordinates (mu +- r + 1/2) s - 1/2 to an integer. */
void oracle_margins(int K, const double *mu, const double *chol, double R2,
                    int H, int W, int out_H, int out_W,
                    double *d2_gap, double *edge_gap)
{
    double sx = (double)out_W / (double)W, sy = (double)out_H / (double)H;
    for (int k = 0; k < K; k++) {
        double r = sqrt(R2 * oracle_lambda_max(chol + 3 * k));
        double mx = mu[2 * k], my = mu[2 * k + 1];
        double e[4] = {(mx - r + 0.5) * sx - 0.5, (mx + r + 0.5) * sx - 0.5,
                       (my - r + 0.5) * sy - 0.5, (my + r + 0.5) * sy - 0.5};
        double eg = 1.0;
        for (int q = 0; q < 4; q++) {
            double f = fabs(e[q] - floor(e[q] + 0.5));
            if (f < eg) eg = f;
        }
        edge_gap[k] = eg;
        int x0 = (int)floor(e[0]) - 1, x1 = (int)ceil(e[1]) + 1;
        int y0 = (int)floor(e[2]) - 1, y1 = (int)ceil(e[3]) + 1;
        if (x0 < 0) x0 = 0;
        if (y0 < 0) y0 = 0;
        if (x1 > out_W - 1) x1 = out_W - 1;
        if (y1 > out_H - 1) y1 = out_H - 1;
        double dg = 1e300;
        for (int i = y0; i <= y1; i++)
            for (int jx = x0; jx <= x1; jx++) {
                double px = (jx + 0.5) * W / out_W - 0.5, py = (i + 0.5) * H / out_H - 0.5;
                double g = fabs(oracle_d2(mu + 2 * k, chol + 3 * k, px, py) - R2);
                if (g < dg) dg = g;
            }
        d2_gap[k] = dg;
    }
}

/* Margin of sample points for sampled parity (SURVEY §8(c) rule P1 applied
 * to samples instead of kernels): for each point x_i, the smallest
 * |d^2_j(x_i) - R2| over EVERY kernel j (dense).  A pixel whose value could
 * depend on a cull decision taken differently in fp32 and fp64 has a small
 * margin; a pixel with margin tau in d^2 is also inside every listing box
 * by at least r tau / (2 R2) px, so box-edge rounding cannot drop a kernel
 * it needs. */
void oracle_point_margins(int K, const double *mu, const double *chol, double R2,
                          int n, const double *xs, const double *ys, double *gap)
{
    for (int i = 0; i < n; i++) {
        double g = 1e300;
        for (int k = 0; k < K; k++) {
            double d = fabs(oracle_d2(mu + 2 * k, chol + 3 * k, xs[i], ys[i]) - R2);
            if (d < g) g = d;
        }
        gap[i] = g;
    }
}
