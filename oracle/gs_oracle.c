/*
 * oracle/gs_oracle.c -- the CPU ORACLE for the gsplat hot path (arXiv 2409.06765).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2409_06765_b200/) never imports, links or executes anything in oracle/,
 * and this file shares no code, header, table or constant generator with it.
 *
 * What it is: a plain, slow, deliberately unblocked implementation of what the
 * method computes, following the paper step by step.  Citations are to
 * /root/reference/PAPER.md by line ("P:534") and to SURVEY.md Appendix A step
 * names (F1..F15, I1..I4, R1..R3, B1..B6, P1..P9), which restate the paper.
 *
 *  - Values and gradients are computed in fp64 (the paper fixes no precision).
 *  - Integer decisions that the GPU takes in fp32 -- radii, the projected mean and
 *    the depth bits that form tile keys -- are taken here in fp32 with the op
 *    order written down in DESIGN.md ("key path", reading Q28), so keys, sort
 *    order and tile ranges can be compared bit-exactly.  Compile with
 *    -ffp-contract=off (no FMA contraction) so every fp32 op rounds once.
 *  - Compositing uses NO tiles as an accelerator: every pixel walks the camera's
 *    whole global depth-sorted visible list ("sorted by depth") and keeps a
 *    splat only if the pixel's 16x16 tile lies inside the splat's 3-sigma tile
 *    rectangle ("include it in a tile bin if its bounding box intersects
 *    with the tile"), which is part of the method's definition.
 *
 * Parity status of each function is stated in DESIGN.md section "Oracle pins".
 * The SH basis (Q22) is pinned, signs included, to the real spherical harmonics built
 * from scipy's complex Y_l^m with the Condon-Shortley phase (tests/test_oracle_pins.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double near_plane;   /* 0.01 : cull iff depth <  near (Q18, pinned by Fig. 1)     */
    double far_plane;    /* 1e10 : cull iff depth >  far                                  */
    double eps2d;        /* 0.3  : low-pass s                                     */
    double alpha_max;    /* 0.99 : opacity saturation (north_star; Q13)                   */
    double alpha_min;    /* 1/255: skip iff alpha < alpha_min (Q14)                       */
    double t_min;        /* 1e-4 : stop iff T*(1-alpha) <= t_min, exclusive (Q15)         */
    double amb_safety;   /* factor on the derived fp32 error bounds of the decisions (Q28b) */
    double amb_rel_floor;/* minimum relative ambiguity margin (FD scene sampling)          */
    int32_t tile_size;   /* 16                                                    */
    int32_t antialiased; /* 0 classic | 1 compensated opacity                 */
    int32_t sh_degree;   /* -1 direct RGB colors | 0..3 spherical harmonics               */
    int32_t bbox_mode;   /* 0 per-axis 3-sigma AABB (Q12) | 1 square 3*sqrt(lambda_max) |
                            2 opacity-aware extent (Q36)                                   */
    int32_t fov_clamp;   /* 1 clamp t_x/t_z, t_y/t_z for J only (Q27)                     */
    int32_t channels;    /* 0: RGB from the projection | D > 0: N-D features,
                            render inputs are [C*N, D] feature rows, images [C,H,W,D]     */
} or_opts;

#define OR_MAX_CH 64
static int n_channels(const or_opts *o) { return o->channels > 0 ? o->channels : 3; }

/* ------------------------------------------------------------------------- */
/* Spherical harmonics, real basis up to degree 3 ([bk]).  */
/* P:505 writes c = SH((mu - t)/||mu - t||); P:476 says colour is SH-encoded.  */
/* ------------------------------------------------------------------------- */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Y[j] for j < (deg+1)^2 at unit direction (x,y,z). */
static void sh_basis(int deg, double x, double y, double z, double *Y)
{
    Y[0] = SH_C0;
    if (deg < 1) return;
    Y[1] = -SH_C1 * y;
    Y[2] = SH_C1 * z;
    Y[3] = -SH_C1 * x;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = SH_C2[0] * x * y;
    Y[5] = SH_C2[1] * y * z;
    Y[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    Y[7] = SH_C2[3] * x * z;
    Y[8] = SH_C2[4] * (xx - yy);
    if (deg < 3) return;
    Y[9]  = SH_C3[0] * y * (3.0 * xx - yy);
    Y[10] = SH_C3[1] * x * y * z;
    Y[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    Y[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    Y[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    Y[14] = SH_C3[5] * z * (xx - yy);
    Y[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

/* dY[j][0..2] = dY_j / d(x,y,z), the partial derivatives of the polynomials above
 * (treating x,y,z as independent; the normalisation is chained separately, P7). */
static void sh_basis_grad(int deg, double x, double y, double z, double dY[16][3])
{
    memset(dY, 0, sizeof(double) * 16 * 3);
    if (deg < 1) return;
    dY[1][1] = -SH_C1;
    dY[2][2] = SH_C1;
    dY[3][0] = -SH_C1;
    if (deg < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    dY[4][0] = SH_C2[0] * y;              dY[4][1] = SH_C2[0] * x;
    dY[5][1] = SH_C2[1] * z;              dY[5][2] = SH_C2[1] * y;
    dY[6][0] = SH_C2[2] * (-2.0 * x);     dY[6][1] = SH_C2[2] * (-2.0 * y);  dY[6][2] = SH_C2[2] * (4.0 * z);
    dY[7][0] = SH_C2[3] * z;              dY[7][2] = SH_C2[3] * x;
    dY[8][0] = SH_C2[4] * (2.0 * x);      dY[8][1] = SH_C2[4] * (-2.0 * y);
    if (deg < 3) return;
    dY[9][0]  = SH_C3[0] * (6.0 * x * y);
    dY[9][1]  = SH_C3[0] * (3.0 * xx - 3.0 * yy);
    dY[10][0] = SH_C3[1] * y * z;  dY[10][1] = SH_C3[1] * x * z;  dY[10][2] = SH_C3[1] * x * y;
    dY[11][0] = SH_C3[2] * (-2.0 * x * y);
    dY[11][1] = SH_C3[2] * (4.0 * zz - xx - 3.0 * yy);
    dY[11][2] = SH_C3[2] * (8.0 * y * z);
    dY[12][0] = SH_C3[3] * (-6.0 * x * z);
    dY[12][1] = SH_C3[3] * (-6.0 * y * z);
    dY[12][2] = SH_C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    dY[13][0] = SH_C3[4] * (4.0 * zz - 3.0 * xx - yy);
    dY[13][1] = SH_C3[4] * (-2.0 * x * y);
    dY[13][2] = SH_C3[4] * (8.0 * x * z);
    dY[14][0] = SH_C3[5] * (2.0 * x * z);
    dY[14][1] = SH_C3[5] * (-2.0 * y * z);
    dY[14][2] = SH_C3[5] * (xx - yy);
    dY[15][0] = SH_C3[6] * (3.0 * xx - 3.0 * yy);
    dY[15][1] = SH_C3[6] * (-6.0 * x * y);
}

/* Tolerance model only (absmode of the projection backward): the same polynomials with
 * every coefficient and monomial taken in magnitude (subtractions become additions), i.e. the
 * scale of the rounding error of evaluating Y_j and dY_j in fp32.  Evaluated at |dir|. */
static void sh_basis_mag(int deg, double x, double y, double z, double *Y, double dY[16][3])
{
    x = fabs(x); y = fabs(y); z = fabs(z);
    memset(dY, 0, sizeof(double) * 16 * 3);
    Y[0] = SH_C0;
    if (deg < 1) return;
    Y[1] = SH_C1 * y; Y[2] = SH_C1 * z; Y[3] = SH_C1 * x;
    dY[1][1] = dY[2][2] = dY[3][0] = SH_C1;
    if (deg < 2) return;
    const double c2 = fabs(SH_C2[0]), c22 = fabs(SH_C2[2]), c24 = fabs(SH_C2[4]);
    double xx = x * x, yy = y * y, zz = z * z;
    Y[4] = c2 * x * y; Y[5] = c2 * y * z; Y[6] = c22 * (2.0 * zz + xx + yy); Y[7] = c2 * x * z;
    Y[8] = c24 * (xx + yy);
    dY[4][0] = c2 * y;  dY[4][1] = c2 * x;
    dY[5][1] = c2 * z;  dY[5][2] = c2 * y;
    dY[6][0] = c22 * 2.0 * x;  dY[6][1] = c22 * 2.0 * y;  dY[6][2] = c22 * 4.0 * z;
    dY[7][0] = c2 * z;  dY[7][2] = c2 * x;
    dY[8][0] = c24 * 2.0 * x;  dY[8][1] = c24 * 2.0 * y;
    if (deg < 3) return;
    double k[7];
    for (int i = 0; i < 7; i++) k[i] = fabs(SH_C3[i]);
    Y[9]  = k[0] * y * (3.0 * xx + yy);
    Y[10] = k[1] * x * y * z;
    Y[11] = k[2] * y * (4.0 * zz + xx + yy);
    Y[12] = k[3] * z * (2.0 * zz + 3.0 * xx + 3.0 * yy);
    Y[13] = k[4] * x * (4.0 * zz + xx + yy);
    Y[14] = k[5] * z * (xx + yy);
    Y[15] = k[6] * x * (xx + 3.0 * yy);
    dY[9][0] = k[0] * 6.0 * x * y;            dY[9][1] = k[0] * (3.0 * xx + 3.0 * yy);
    dY[10][0] = k[1] * y * z;  dY[10][1] = k[1] * x * z;  dY[10][2] = k[1] * x * y;
    dY[11][0] = k[2] * 2.0 * x * y;  dY[11][1] = k[2] * (4.0 * zz + xx + 3.0 * yy);  dY[11][2] = k[2] * 8.0 * y * z;
    dY[12][0] = k[3] * 6.0 * x * z;  dY[12][1] = k[3] * 6.0 * y * z;  dY[12][2] = k[3] * (6.0 * zz + 3.0 * xx + 3.0 * yy);
    dY[13][0] = k[4] * (4.0 * zz + 3.0 * xx + yy);  dY[13][1] = k[4] * 2.0 * x * y;  dY[13][2] = k[4] * 8.0 * x * z;
    dY[14][0] = k[5] * 2.0 * x * z;  dY[14][1] = k[5] * 2.0 * y * z;  dY[14][2] = k[5] * (xx + yy);
    dY[15][0] = k[6] * (3.0 * xx + 3.0 * yy);  dY[15][1] = k[6] * 6.0 * x * y;
}

/* exported for the quadrature / FD pins */
void or_sh_basis(int32_t deg, double x, double y, double z, double *Y) { sh_basis(deg, x, y, z, Y); }
void or_sh_basis_grad(int32_t deg, double x, double y, double z, double *dY)
{
    double g[16][3];
    sh_basis_grad(deg, x, y, z, g);
    memcpy(dY, g, sizeof g);
}

/* ------------------------------------------------------------------------- */
/* F1: quaternion (w,x,y,z), Hamilton, to rotation matrix.          */
/* ------------------------------------------------------------------------- */
static void quat_to_rot(double w, double x, double y, double z, double R[3][3])
{
    R[0][0] = 1.0 - 2.0 * (y * y + z * z);
    R[0][1] = 2.0 * (x * y - w * z);
    R[0][2] = 2.0 * (x * z + w * y);
    R[1][0] = 2.0 * (x * y + w * z);
    R[1][1] = 1.0 - 2.0 * (x * x + z * z);
    R[1][2] = 2.0 * (y * z - w * x);
    R[2][0] = 2.0 * (x * z - w * y);
    R[2][1] = 2.0 * (y * z + w * x);
    R[2][2] = 1.0 - 2.0 * (x * x + y * y);
}

void or_quat_to_rotmat(const double *q, double *R9)
{
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    double R[3][3];
    quat_to_rot(q[0] / n, q[1] / n, q[2] / n, q[3] / n, R);
    memcpy(R9, R, sizeof R);
}

/* ------------------------------------------------------------------------- */
/* Key path: fp32, fixed op order (reading Q28).  Produces radii,   */
/* the fp32 projected mean and depth; decides visibility (F4, F9, F12, F13).  */
/* Every expression below is one IEEE op per operator, left to right.         */
/* ------------------------------------------------------------------------- */
typedef struct {
    int   visible;
    int   rx, ry;
    float mx, my, depth;
    /* fp32 evaluation of F10 / F15 (the conic and o_eff): sizes the ambiguity margin of the
     * threshold decisions (Q28b); decides nothing */
    float conic[3], opac;
} keypath_t;

static keypath_t key_path_f32(const or_opts *o, int W, int H, const float *mu, const float *q,
                              const float *s, float op, const float *vm /*4x4*/, const float *Kc /*3x3*/)
{
    keypath_t kp = {0, 0, 0, 0.f, 0.f, 0.f, {0.f, 0.f, 0.f}, 0.f};
    /* KP1 (F3): t = W mu + w */
    float tx = ((vm[0] * mu[0] + vm[1] * mu[1]) + vm[2] * mu[2]) + vm[3];
    float ty = ((vm[4] * mu[0] + vm[5] * mu[1]) + vm[6] * mu[2]) + vm[7];
    float tz = ((vm[8] * mu[0] + vm[9] * mu[1]) + vm[10] * mu[2]) + vm[11];
    /* KP2 (F4): depth, near/far (strict, Q18) */
    if (!(tz >= (float)o->near_plane) || tz > (float)o->far_plane) return kp;
    /* KP3 (F1): q_hat = q / ||q|| */
    float qn2 = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
    if (!(qn2 > 0.f) || !isfinite(qn2)) return kp;
    float qn = sqrtf(qn2);
    float w = q[0] / qn, x = q[1] / qn, y = q[2] / qn, z = q[3] / qn;
    /* KP4 (F1): R(q_hat) */
    float R[3][3];
    R[0][0] = 1.f - 2.f * (y * y + z * z);
    R[0][1] = 2.f * (x * y - w * z);
    R[0][2] = 2.f * (x * z + w * y);
    R[1][0] = 2.f * (x * y + w * z);
    R[1][1] = 1.f - 2.f * (x * x + z * z);
    R[1][2] = 2.f * (y * z - w * x);
    R[2][0] = 2.f * (x * z - w * y);
    R[2][1] = 2.f * (y * z + w * x);
    R[2][2] = 1.f - 2.f * (x * x + y * y);
    /* KP5 (F2): M = R diag(s) ; KP6: Sigma = M M^T */
    float M[3][3], S[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[i][j] = R[i][j] * s[j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) S[i][j] = (M[i][0] * M[j][0] + M[i][1] * M[j][1]) + M[i][2] * M[j][2];
    /* KP7 (F5): Sigma_c = Wr Sigma Wr^T, via A = Wr Sigma */
    float Wr[3][3] = {{vm[0], vm[1], vm[2]}, {vm[4], vm[5], vm[6]}, {vm[8], vm[9], vm[10]}};
    float A[3][3], Sc[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) A[i][j] = (Wr[i][0] * S[0][j] + Wr[i][1] * S[1][j]) + Wr[i][2] * S[2][j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) Sc[i][j] = (A[i][0] * Wr[j][0] + A[i][1] * Wr[j][1]) + A[i][2] * Wr[j][2];
    /* KP8 (F6): J with focals (Q4) and optional frustum clamp (Q27) */
    float fx = Kc[0], fy = Kc[4], cx = Kc[2], cy = Kc[5];
    float txc = tx, tyc = ty;
    if (o->fov_clamp) {
        float tanx = (0.5f * (float)W) / fx, tany = (0.5f * (float)H) / fy;
        float lxp = ((float)W - cx) / fx + 0.3f * tanx, lxn = cx / fx + 0.3f * tanx;
        float lyp = ((float)H - cy) / fy + 0.3f * tany, lyn = cy / fy + 0.3f * tany;
        float u = tx / tz, v = ty / tz;
        float uc = fminf(lxp, fmaxf(-lxn, u)), vc = fminf(lyp, fmaxf(-lyn, v));
        txc = tz * uc;
        tyc = tz * vc;
    }
    float J[2][3];
    J[0][0] = fx / tz; J[0][1] = 0.f; J[0][2] = -(fx * txc) / (tz * tz);
    J[1][0] = 0.f; J[1][1] = fy / tz; J[1][2] = -(fy * tyc) / (tz * tz);
    /* KP9 (F7): Sigma' = J Sigma_c J^T via B = J Sigma_c */
    float B[2][3], Sp[2][2];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 3; j++) B[i][j] = (J[i][0] * Sc[0][j] + J[i][1] * Sc[1][j]) + J[i][2] * Sc[2][j];
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++) Sp[i][j] = (B[i][0] * J[j][0] + B[i][1] * J[j][1]) + B[i][2] * J[j][2];
    /* KP10 (F8): low-pass */
    float a = Sp[0][0] + (float)o->eps2d, b = Sp[0][1], c = Sp[1][1] + (float)o->eps2d;
    /* KP11 (F9): det */
    float det = a * c - b * b;
    if (!(det > 0.f)) return kp;
    /* KP12 (F12): radii */
    int rx, ry;
    if (o->bbox_mode == 0 || o->bbox_mode == 2) {
        rx = (int)ceilf(3.f * sqrtf(a));
        ry = (int)ceilf(3.f * sqrtf(c));
        if (o->bbox_mode == 2 && o->alpha_min > 0.0) {
            /* KP12b (DESIGN Q36): opacity-aware extent, fp32.
             * A splat reaches alpha >= alpha_min only where sigma <= tau = ln(o_eff/alpha_min)
             * (R1: alpha = o_eff exp(-sigma)).  Upper bound: x = o_eff/alpha_min = m 2^e,
             * ln x = e ln2 + ln m and ln m <= 2(m-1)/(m+1) for m in (0,1].  Mahalanobis
             * radius^2 = 2 tau (sigma = d^T conic d / 2), with the fp32 margin 1.004, 4e-3. */
            float comp_b = 1.f;
            if (o->antialiased) {
                float det_raw_b = Sp[0][0] * Sp[1][1] - Sp[0][1] * Sp[0][1];
                comp_b = sqrtf(fmaxf(0.f, det_raw_b / det));
            }
            float o_eff = op * comp_b;
            float amin = (float)o->alpha_min;
            if (!(o_eff >= amin)) return kp;               /* alpha < alpha_min at every pixel */
            int e;
            float m = frexpf(o_eff / amin, &e);
            float tau_ub = (float)e * 0.693147182f + (2.f * (m - 1.f)) / (m + 1.f);
            float k2 = 2.f * (tau_ub * 1.004f + 4e-3f);
            float cond = (a * c) / det;                    /* 1/(1-rho^2) of Sigma'+sI */
            if (k2 < 9.f && cond <= 1000.f) {              /* else the 3-sigma extent */
                rx = (int)ceilf(sqrtf(k2 * a));
                ry = (int)ceilf(sqrtf(k2 * c));
            }
        }
    } else {
        float m = 0.5f * (a + c);
        float lam = m + sqrtf(fmaxf(0.f, m * m - det));
        rx = ry = (int)ceilf(3.f * sqrtf(lam));
    }
    /* KP13 (F11): mu' = f t/t_z + c */
    float mx = (fx * tx) / tz + cx;
    float my = (fy * ty) / tz + cy;
    /* KP14 (F13): off-screen cull (Q19) */
    if (mx + (float)rx <= 0.f || mx - (float)rx >= (float)W || my + (float)ry <= 0.f ||
        my - (float)ry >= (float)H)
        return kp;
    if (!isfinite(mx) || !isfinite(my)) return kp;
    kp.visible = 1; kp.rx = rx; kp.ry = ry; kp.mx = mx; kp.my = my; kp.depth = tz;
    /* KP15 (F9, F10, F15 in fp32): conic and effective opacity, for the error bound of Q28b */
    kp.conic[0] = c / det;
    kp.conic[1] = -b / det;
    kp.conic[2] = a / det;
    float comp = 1.f;
    if (o->antialiased) {
        float det_raw = Sp[0][0] * Sp[1][1] - Sp[0][1] * Sp[0][1];
        comp = sqrtf(fmaxf(0.f, det_raw / det));
    }
    kp.opac = op * comp;
    return kp;
}

/* I1 (Q20): tile rectangle [x0,x1) x [y0,y1) in fp32, /tile is exact. */
static void tile_rect(int tile, int TX, int TY, float mx, float my, int rx, int ry,
                      int *x0, int *x1, int *y0, int *y1)
{
    float ft = (float)tile;
    int a0 = (int)floorf((mx - (float)rx) / ft), a1 = (int)ceilf((mx + (float)rx) / ft);
    int b0 = (int)floorf((my - (float)ry) / ft), b1 = (int)ceilf((my + (float)ry) / ft);
    *x0 = a0 < 0 ? 0 : (a0 > TX ? TX : a0);
    *x1 = a1 < 0 ? 0 : (a1 > TX ? TX : a1);
    *y0 = b0 < 0 ? 0 : (b0 > TY ? TY : b0);
    *y1 = b1 < 0 ? 0 : (b1 > TY ? TY : b1);
}

/* ------------------------------------------------------------------------- */
/* fp64 values path, F1..F15, for one (c,n).                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    /* inputs promoted */
    double mu[3], qraw[4], qn, qh[4], s[3], o;
    double Wr[3][3], w[3], fx, fy, cx, cy;
    /* intermediates */
    double R[3][3], M[3][3], Sig[3][3], t[3], Sc[3][3];
    double u, v, uc, vc, txc, tyc;
    int clamp_x, clamp_y;
    double J[2][3], Sp[2][2], Spb[2][2], det, detb, comp;
    double conic[3];
    double mean2d[2];
    double campos[3], e[3], enorm, dir[3];
    double raw[3], rgb[3];
    double rawabs[3];   /* 0.5 + sum_j |Y_j sh_j|: scale of the fp32 rounding of raw (tolerance) */
    double opac_eff;
} proj64_t;

static void project64(const or_opts *o, int W, int H, const float *mu, const float *q, const float *s,
                      float op, const float *colors, int K, const float *vm, const float *Kc, proj64_t *P)
{
    for (int i = 0; i < 3; i++) P->mu[i] = mu[i], P->s[i] = s[i];
    for (int i = 0; i < 4; i++) P->qraw[i] = q[i];
    P->o = op;
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) P->Wr[i][j] = vm[4 * i + j];
        P->w[i] = vm[4 * i + 3];
    }
    P->fx = Kc[0]; P->fy = Kc[4]; P->cx = Kc[2]; P->cy = Kc[5];
    /* F1 */
    P->qn = sqrt(P->qraw[0] * P->qraw[0] + P->qraw[1] * P->qraw[1] + P->qraw[2] * P->qraw[2] +
                 P->qraw[3] * P->qraw[3]);
    for (int i = 0; i < 4; i++) P->qh[i] = P->qraw[i] / P->qn;
    quat_to_rot(P->qh[0], P->qh[1], P->qh[2], P->qh[3], P->R);
    /* F2: M = R S, Sigma = M M^T */
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) P->M[i][j] = P->R[i][j] * P->s[j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc += P->M[i][k] * P->M[j][k];
            P->Sig[i][j] = acc;
        }
    /* F3: t = W mu + w ("t = T_cw q") */
    for (int i = 0; i < 3; i++) {
        double acc = P->w[i];
        for (int k = 0; k < 3; k++) acc += P->Wr[i][k] * P->mu[k];
        P->t[i] = acc;
    }
    /* F5: Sigma_c = W Sigma W^T (Fig. P:423) */
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double acc = 0;
            for (int k = 0; k < 3; k++)
                for (int l = 0; l < 3; l++) acc += P->Wr[i][k] * P->Sig[k][l] * P->Wr[j][l];
            P->Sc[i][j] = acc;
        }
    /* F6: J (P:695-709 with focals; Q4) with frustum clamp for J only (Q27) */
    double tz = P->t[2];
    P->u = P->t[0] / tz; P->v = P->t[1] / tz;
    P->uc = P->u; P->vc = P->v; P->clamp_x = P->clamp_y = 0;
    if (o->fov_clamp) {
        double tanx = 0.5 * W / P->fx, tany = 0.5 * H / P->fy;
        double lxp = (W - P->cx) / P->fx + 0.3 * tanx, lxn = P->cx / P->fx + 0.3 * tanx;
        double lyp = (H - P->cy) / P->fy + 0.3 * tany, lyn = P->cy / P->fy + 0.3 * tany;
        if (P->u > lxp) { P->uc = lxp; P->clamp_x = 1; }
        if (P->u < -lxn) { P->uc = -lxn; P->clamp_x = 1; }
        if (P->v > lyp) { P->vc = lyp; P->clamp_y = 1; }
        if (P->v < -lyn) { P->vc = -lyn; P->clamp_y = 1; }
    }
    P->txc = tz * P->uc; P->tyc = tz * P->vc;
    P->J[0][0] = P->fx / tz; P->J[0][1] = 0; P->J[0][2] = -P->fx * P->txc / (tz * tz);
    P->J[1][0] = 0; P->J[1][1] = P->fy / tz; P->J[1][2] = -P->fy * P->tyc / (tz * tz);
    /* F7: Sigma' = J Sigma_c J^T */
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 2; j++) {
            double acc = 0;
            for (int k = 0; k < 3; k++)
                for (int l = 0; l < 3; l++) acc += P->J[i][k] * P->Sc[k][l] * P->J[j][l];
            P->Sp[i][j] = acc;
        }
    /* F8: + s I in both modes (Q6) */
    P->Spb[0][0] = P->Sp[0][0] + o->eps2d; P->Spb[0][1] = P->Sp[0][1];
    P->Spb[1][0] = P->Sp[1][0];            P->Spb[1][1] = P->Sp[1][1] + o->eps2d;
    /* F9: determinants and the A.4 compensation (Q7) */
    P->det = P->Sp[0][0] * P->Sp[1][1] - P->Sp[0][1] * P->Sp[1][0];
    P->detb = P->Spb[0][0] * P->Spb[1][1] - P->Spb[0][1] * P->Spb[1][0];
    if (o->antialiased) {
        double r = P->det / P->detb;
        P->comp = sqrt(r > 0 ? r : 0);
    } else {
        P->comp = 1.0;
    }
    /* F10: conic = (Sigma'+sI)^-1 packed (A, B, C) */
    P->conic[0] = P->Spb[1][1] / P->detb;
    P->conic[1] = -P->Spb[0][1] / P->detb;
    P->conic[2] = P->Spb[0][0] / P->detb;
    /* F11: P:790-791 */
    P->mean2d[0] = P->fx * P->t[0] / tz + P->cx;
    P->mean2d[1] = P->fy * P->t[1] / tz + P->cy;
    /* F14: colour (SH basis [bk], Q22) */
    if (o->sh_degree >= 0) {
        /* campos = -Wr^T w */
        for (int i = 0; i < 3; i++) {
            double acc = 0;
            for (int k = 0; k < 3; k++) acc -= P->Wr[k][i] * P->w[k];
            P->campos[i] = acc;
        }
        for (int i = 0; i < 3; i++) P->e[i] = P->mu[i] - P->campos[i];
        P->enorm = sqrt(P->e[0] * P->e[0] + P->e[1] * P->e[1] + P->e[2] * P->e[2]);
        for (int i = 0; i < 3; i++) P->dir[i] = P->e[i] / P->enorm;
        double Y[16];
        int nb = (o->sh_degree + 1) * (o->sh_degree + 1);
        sh_basis(o->sh_degree, P->dir[0], P->dir[1], P->dir[2], Y);
        for (int ch = 0; ch < 3; ch++) {
            double acc = 0.5, aa = 0.5;
            for (int j = 0; j < nb; j++) {
                acc += Y[j] * (double)colors[(int64_t)j * 3 + ch];
                aa += fabs(Y[j] * (double)colors[(int64_t)j * 3 + ch]);
            }
            P->raw[ch] = acc;
            P->rawabs[ch] = aa;
            P->rgb[ch] = acc > 0 ? acc : 0;
        }
    } else {
        for (int ch = 0; ch < 3; ch++) {
            P->raw[ch] = P->rgb[ch] = colors[ch];
            P->rawabs[ch] = 0;
        }
    }
    (void)K;
    /* F15 */
    P->opac_eff = P->o * P->comp;
}

/* Magnitudes of every forward quantity the projection backward uses (absmode of
 * or_project_bwd; a tolerance model, not a result). */
static void abs_proj(proj64_t *P)
{
    double *blocks[] = {&P->mu[0], &P->R[0][0], &P->M[0][0], &P->Sig[0][0], &P->t[0], &P->Sc[0][0],
                        &P->J[0][0], &P->Sp[0][0], &P->Spb[0][0], &P->conic[0], &P->campos[0], &P->e[0],
                        &P->dir[0], &P->Wr[0][0], &P->w[0], &P->qh[0], &P->s[0]};
    int sizes[] = {3, 9, 9, 9, 3, 9, 6, 4, 4, 3, 3, 3, 3, 9, 3, 4, 3};
    for (int b = 0; b < (int)(sizeof sizes / sizeof sizes[0]); b++)
        for (int i = 0; i < sizes[b]; i++) blocks[b][i] = fabs(blocks[b][i]);
    P->txc = fabs(P->txc); P->tyc = fabs(P->tyc);
    P->fx = fabs(P->fx); P->fy = fabs(P->fy);
    /* raw keeps its sign: it only selects the unclamped SH channels (P7); det > 0 as well */
}

/* ------------------------------------------------------------------------- */
/* Exported: projection over all (c, n).                                       */
/* ------------------------------------------------------------------------- */
int or_project(const or_opts *o, int64_t N, int32_t C, int32_t W, int32_t H, const float *means,
               const float *quats, const float *scales, const float *opacities, const float *colors,
               int32_t K, const float *viewmats, const float *Ks,
               int32_t *radii, float *mean2d_f, float *depth_f, float *dec,
               double *mean2d, double *depth, double *conic, double *comp, double *opac_eff, double *rgb)
{
    int64_t stride = o->sh_degree >= 0 ? (int64_t)K * 3 : 3;
#pragma omp parallel for schedule(static)
    for (int64_t idx = 0; idx < (int64_t)C * N; idx++) {
        int64_t c = idx / N, n = idx % N;
        const float *vm = viewmats + 16 * c, *Kc = Ks + 9 * c;
        keypath_t kp = key_path_f32(o, W, H, means + 3 * n, quats + 4 * n, scales + 3 * n, opacities[n], vm, Kc);
        for (int i = 0; i < 3; i++) dec[4 * idx + i] = kp.visible ? kp.conic[i] : 0.f;
        dec[4 * idx + 3] = kp.visible ? kp.opac : 0.f;
        radii[2 * idx] = kp.visible ? kp.rx : 0;
        radii[2 * idx + 1] = kp.visible ? kp.ry : 0;
        mean2d_f[2 * idx] = kp.visible ? kp.mx : 0.f;
        mean2d_f[2 * idx + 1] = kp.visible ? kp.my : 0.f;
        depth_f[idx] = kp.visible ? kp.depth : 0.f;
        if (!kp.visible) {
            mean2d[2 * idx] = mean2d[2 * idx + 1] = 0;
            depth[idx] = 0; conic[3 * idx] = conic[3 * idx + 1] = conic[3 * idx + 2] = 0;
            comp[idx] = 0; opac_eff[idx] = 0; rgb[3 * idx] = rgb[3 * idx + 1] = rgb[3 * idx + 2] = 0;
            continue;
        }
        proj64_t P;
        project64(o, W, H, means + 3 * n, quats + 4 * n, scales + 3 * n, opacities[n], colors + stride * n,
                  K, vm, Kc, &P);
        mean2d[2 * idx] = P.mean2d[0]; mean2d[2 * idx + 1] = P.mean2d[1];
        depth[idx] = P.t[2];
        for (int i = 0; i < 3; i++) conic[3 * idx + i] = P.conic[i], rgb[3 * idx + i] = P.rgb[i];
        comp[idx] = P.comp;
        opac_eff[idx] = P.opac_eff;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* I1-I4 by brute force: enumerate every (c, n, tile) with the tile inside the */
/* rectangle, key = (c << (32+B)) | (tile << 32) | bits(depth),    */
/* value = c*N + n, then sort by (key, value) and take lower bounds.           */
/* Returns M; writes outputs only when M <= cap.                               */
/* ------------------------------------------------------------------------- */
typedef struct { uint64_t key; int32_t id; } kv_t;
static int kv_cmp(const void *a, const void *b)
{
    const kv_t *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int tile_bits(int ntiles)
{
    int B = 0;
    while ((1LL << B) < ntiles) B++;
    return B;
}

int64_t or_isect(const or_opts *o, int32_t C, int64_t N, int32_t W, int32_t H, const int32_t *radii,
                 const float *mean2d_f, const float *depth_f, int64_t cap, uint64_t *keys, int32_t *ids,
                 int32_t *tile_offsets)
{
    int T = o->tile_size, TX = (W + T - 1) / T, TY = (H + T - 1) / T;
    int B = tile_bits(TX * TY);
    int64_t M = 0;
    for (int64_t idx = 0; idx < (int64_t)C * N; idx++) {
        if (radii[2 * idx] <= 0 || radii[2 * idx + 1] <= 0) continue;
        int x0, x1, y0, y1;
        tile_rect(T, TX, TY, mean2d_f[2 * idx], mean2d_f[2 * idx + 1], radii[2 * idx], radii[2 * idx + 1],
                  &x0, &x1, &y0, &y1);
        M += (int64_t)(x1 - x0) * (y1 - y0);
    }
    if (M > cap) return M;
    kv_t *kv = (kv_t *)malloc(sizeof(kv_t) * (M > 0 ? M : 1));
    int64_t m = 0;
    for (int64_t idx = 0; idx < (int64_t)C * N; idx++) {
        if (radii[2 * idx] <= 0 || radii[2 * idx + 1] <= 0) continue;
        int64_t c = idx / N;
        int x0, x1, y0, y1;
        tile_rect(T, TX, TY, mean2d_f[2 * idx], mean2d_f[2 * idx + 1], radii[2 * idx], radii[2 * idx + 1],
                  &x0, &x1, &y0, &y1);
        uint32_t dbits;
        memcpy(&dbits, &depth_f[idx], 4);
        for (int ty = y0; ty < y1; ty++)
            for (int tx = x0; tx < x1; tx++) {
                uint64_t tile = (uint64_t)(ty * TX + tx);
                kv[m].key = ((uint64_t)c << (32 + B)) | (tile << 32) | (uint64_t)dbits;
                kv[m].id = (int32_t)idx;
                m++;
            }
    }
    qsort(kv, M, sizeof(kv_t), kv_cmp);
    for (int64_t i = 0; i < M; i++) keys[i] = kv[i].key, ids[i] = kv[i].id;
    /* I4: offsets[c*TT + t] = first index whose (cam, tile) >= (c, t); offsets[end] = M */
    int64_t ntot = (int64_t)C * TX * TY;
    int64_t k = 0;
    for (int64_t bin = 0; bin < ntot; bin++) {
        int64_t c = bin / (TX * TY), t = bin % (TX * TY);
        uint64_t lo = ((uint64_t)c << (32 + B)) | ((uint64_t)t << 32);
        while (k < M && keys[k] < lo) k++;
        tile_offsets[bin] = (int32_t)k;
    }
    tile_offsets[ntot] = (int32_t)M;
    free(kv);
    return M;
}

/* ------------------------------------------------------------------------- */
/* Rendering.  Per camera: the visible set sorted by (fp32 depth bits, n)      */
/* ("sorts them per tile by depth"; tie-break Q16).                      */
/* ------------------------------------------------------------------------- */
typedef struct { uint32_t dbits; int32_t n; } dn_t;
static int dn_cmp(const void *a, const void *b)
{
    const dn_t *x = a, *y = b;
    if (x->dbits != y->dbits) return x->dbits < y->dbits ? -1 : 1;
    return (x->n > y->n) - (x->n < y->n);
}

typedef struct {
    int64_t count;       /* visible splats of this camera */
    int32_t *n;          /* sorted Gaussian indices */
    int32_t *rect;       /* [count][4] tile rectangle x0,x1,y0,y1 */
} camlist_t;

static void build_camlist(const or_opts *o, int64_t c, int64_t N, int W, int H, const int32_t *radii,
                          const float *mean2d_f, const float *depth_f, camlist_t *L)
{
    int T = o->tile_size, TX = (W + T - 1) / T, TY = (H + T - 1) / T;
    int64_t cnt = 0;
    for (int64_t n = 0; n < N; n++)
        if (radii[2 * (c * N + n)] > 0 && radii[2 * (c * N + n) + 1] > 0) cnt++;
    dn_t *tmp = (dn_t *)malloc(sizeof(dn_t) * (cnt > 0 ? cnt : 1));
    int64_t m = 0;
    for (int64_t n = 0; n < N; n++) {
        int64_t idx = c * N + n;
        if (radii[2 * idx] > 0 && radii[2 * idx + 1] > 0) {
            memcpy(&tmp[m].dbits, &depth_f[idx], 4);
            tmp[m].n = (int32_t)n;
            m++;
        }
    }
    qsort(tmp, cnt, sizeof(dn_t), dn_cmp);
    L->count = cnt;
    L->n = (int32_t *)malloc(sizeof(int32_t) * (cnt > 0 ? cnt : 1));
    L->rect = (int32_t *)malloc(sizeof(int32_t) * 4 * (cnt > 0 ? cnt : 1));
    for (int64_t i = 0; i < cnt; i++) {
        int64_t idx = c * N + tmp[i].n;
        L->n[i] = tmp[i].n;
        tile_rect(T, TX, TY, mean2d_f[2 * idx], mean2d_f[2 * idx + 1], radii[2 * idx], radii[2 * idx + 1],
                  &L->rect[4 * i], &L->rect[4 * i + 1], &L->rect[4 * i + 2], &L->rect[4 * i + 3]);
    }
    free(tmp);
}

static void free_camlist(camlist_t *L)
{
    free(L->n);
    free(L->rect);
}

/* One pixel's forward walk, R1-R3.  Optionally records the composited
 * sequence (index into the camera list, alpha, T before, G, sigma) for B1-B6. */
typedef struct {
    int64_t li;      /* list index */
    double alpha, T, G, sigma, dx, dy;
    int clamped;     /* alpha saturated at alpha_max (decision path) */
    int amb_clamp;   /* that decision was ambiguous: both B6 outcomes are correct (tolerance) */
    double delta;    /* 1 ulp of the fp32 mu' the kernel works with (tolerance model only) */
    double qd;       /* first-order relative change of alpha for a delta shift of mu' */
} contrib_t;

typedef struct {
    double eT;       /* sum over composited splats of alpha qd / (1 - alpha) (tolerance model) */
    double rT;       /* relative fp32 error bound of the final T (decision path, tolerance model) */
    double rgb[OR_MAX_CH], T;
    double dacc;      /* accumulated depth sum z alpha T (App. depth rendering) */
    int64_t last_li;  /* -1 if none */
    int64_t end_li;   /* exclusive end of the evaluated part of the list */
    int ambig;        /* number of ambiguous decisions met on the walk */
    int64_t ncontrib;
} pixres_t;

/* Decision path (reading Q28b).  The three threshold decisions of R2 -- skip when
 * alpha < alpha_min (Q14), saturate at alpha_max (Q13), stop when T(1-alpha) <= t_min
 * (Q15) -- decide an integer (which splats a pixel composites).  They are taken with the
 * paper's formulas evaluated in fp64: sigma = 1/2 (A dx^2 + C dy^2) + B dx dy,
 * alpha = min(alpha_max, o_eff e^-sigma), T(1-alpha) -- on the projected
 * geometry the method works with, i.e. the fp32 projection (as for the tile keys, Q28):
 * mu' from the fp32 key path and the conic (F10) and o_eff (F15) evaluated in fp32 by
 * key_path_f32.  (Taking the fp64 geometry instead moves sigma by |grad sigma| |mu'_f32 -
 * mu'_f64| ~ 1e-4 for a 1-px splat at x ~ 1000 px, and 1.4 % of the pixels of configs[1]
 * would hold a decision that the fp32 projection and the fp64 one take differently.)
 * A pixel is flagged AMBIGUOUS when a decision lies within the error bound of evaluating
 * the same formulas in fp32 (the kernel's precision) instead of fp64.  First-order bound,
 * u = 2^-24, for sigma as a sum of the three terms t_A = 1/2 A dx^2, t_C = 1/2 C dy^2,
 * t_B = B dx dy, s_abs = |t_A| + |t_C| + |t_B|:
 *   each offset dx = fl(mu'_x - p_x) carries u, its square or product 3u, the coefficient
 *   (the conic scaled by a constant) 1.5u, the product with it u: <= 5.5u per term;
 *   the two sums 2u s_abs; in all E_sigma = 8u s_abs (the oracle's fp32 conic, F10, is
 *   the one the kernel is given: tests assert it bit-exact);
 *   r_alpha = E_sigma + 2^-22 + 2u   relative bound on alpha: ex2.approx.f32 (relative
 *             error <= 2^-22, measured on B200 by tools/ubench.cu), the product o_eff G
 *             and the fp32 constant;
 *   r_T     = sum over the composited splats so far of alpha r_alpha / (1 - alpha) + 2u per
 *             step (relative bound on T(1-alpha), a product of fp32 factors 1 - alpha);
 *   ambiguous iff  sigma <= S E_sigma                    (the rounding guard "skip iff sigma < 0")
 *             or   |o_eff e^-sigma - alpha_max| <= S r_alpha alpha_max
 *             or   |alpha - alpha_min|          <= S r_alpha alpha_min
 *             or   |T(1-alpha) - t_min|         <= S r_T t_min
 *   with S = amb_safety (1.5 by default: second-order terms) and every relative margin at
 *   least amb_rel_floor (0 by default; the FD scene sampler asks for 2e-3).
 * The thresholds are the method's constants in fp64; the kernel is given their fp32
 * roundings, a relative change <= u that the 2u terms cover.  The VALUES (colours, T,
 * gradients) stay fp64 on the fp64 projection. */
typedef struct {
    double sigma, dx, dy;   /* fp64 evaluation on the fp32 projected geometry */
    double raw;             /* o_eff e^-sigma */
    double E_sigma;         /* error bound of an fp32 evaluation of sigma */
    double r_alpha;         /* relative error bound of an fp32 evaluation of alpha */
} pairdec_t;

static const double OR_U = 5.9604644775390625e-08;   /* 2^-24 */

static pairdec_t pair_decision(const float *dec4, const float *m2f, double px, double py)
{
    pairdec_t d;
    const double A = dec4[0], B = dec4[1], Cc = dec4[2], o_eff = dec4[3];
    d.dx = (double)m2f[0] - px;                                  /* Delta = mu' - p (Q21) */
    d.dy = (double)m2f[1] - py;
    d.sigma = 0.5 * (A * d.dx * d.dx + Cc * d.dy * d.dy) + B * d.dx * d.dy;
    d.raw = o_eff * exp(-d.sigma);
    double adx = fabs(d.dx), ady = fabs(d.dy);
    double s_abs = 0.5 * fabs(A) * adx * adx + 0.5 * fabs(Cc) * ady * ady + fabs(B) * adx * ady;
    d.E_sigma = 8 * OR_U * s_abs;
    d.r_alpha = d.E_sigma + ldexp(1.0, -22) + 2 * OR_U;
    return d;
}

static int near_thr(double v, double thr, double rel, const or_opts *o)
{
    double m = o->amb_safety * rel;
    if (m < o->amb_rel_floor) m = o->amb_rel_floor;
    return fabs(v - thr) <= m * thr;
}

/* An ambiguous decision admits both outcomes.  flip selects the alternative outcome: bit j
 * set takes the other branch at the j-th ambiguous decision met on the walk (so the walk
 * after a flip is the one a kernel taking that branch follows).  flip = 0 is the fp64
 * decision everywhere.  Returns the decision to take. */
static int decide(int outcome, int ambiguous, uint32_t flip, pixres_t *r)
{
    if (!ambiguous) return outcome;
    int j = r->ambig++;
    return (j < 32 && ((flip >> j) & 1u)) ? !outcome : outcome;
}

static pixres_t pixel_forward(const or_opts *o, const camlist_t *L, int64_t c, int64_t N, int px, int py,
                              const float *mean2d_f, const float *dec, const double *mean2d,
                              const double *conic, const double *opac_eff, const double *rgb,
                              const double *depth, contrib_t *rec, int64_t rec_cap, uint32_t flip)
{
    pixres_t r;
    memset(&r, 0, sizeof r);
    r.T = 1.0; r.last_li = -1; r.end_li = L->count;
    const int D = n_channels(o);
    int tx = px / o->tile_size, ty = py / o->tile_size;
    double p[2] = {px + 0.5, py + 0.5};            /* R1: pixel centre */
    const double amax = o->alpha_max, amin = o->alpha_min, tmin = o->t_min;
    double T = 1.0, rT = 0.0;
    double Tdec = 1.0;   /* transmittance of the decision path: product of the decision alphas */
    for (int64_t i = 0; i < L->count; i++) {
        const int32_t *rc = &L->rect[4 * i];
        if (tx < rc[0] || tx >= rc[1] || ty < rc[2] || ty >= rc[3]) continue;   /* tile predicate */
        int64_t g = c * N + L->n[i];
        const double *Y = &conic[3 * g];
        pairdec_t pd = pair_decision(&dec[4 * g], &mean2d_f[2 * g], p[0], p[1]);
        /* rounding guard of Q14: an fp32 sigma may come out negative near sigma = 0 */
        if (decide(pd.sigma < 0, pd.sigma <= o->amb_safety * pd.E_sigma, flip, &r)) continue;   /* Q14 */
        const int amb_clamp = near_thr(pd.raw, amax, pd.r_alpha, o);
        int clamped = decide(!(pd.raw < amax), amb_clamp, flip, &r);                               /* Q13, Q24 */
        double alpha = clamped ? amax : pd.raw;
        if (decide(alpha < amin, !clamped && near_thr(alpha, amin, pd.r_alpha, o), flip, &r)) continue;  /* Q14 */
        double nT = Tdec * (1.0 - alpha);
        double rT_next = rT + alpha * (clamped ? 2 * OR_U : pd.r_alpha) / (1.0 - alpha) + 2 * OR_U;
        if (decide(nT <= tmin, near_thr(nT, tmin, rT_next, o), flip, &r)) { r.end_li = i + 1; break; }  /* Q15 */
        Tdec = nT;
        /* values (fp64 projection): Delta, sigma, G; alpha = o_eff G unless clamped */
        double dx = mean2d[2 * g] - p[0], dy = mean2d[2 * g + 1] - p[1];
        double sigma = 0.5 * (Y[0] * dx * dx + Y[2] * dy * dy) + Y[1] * dx * dy;
        double G = exp(-sigma);
        alpha = clamped ? amax : opac_eff[g] * G;
        nT = T * (1.0 - alpha);
        /* tolerance model only (not part of the result): 1 ulp of the fp32 mu' */
        double mm = fabs(mean2d[2 * g]) > fabs(mean2d[2 * g + 1]) ? fabs(mean2d[2 * g]) : fabs(mean2d[2 * g + 1]);
        double delta = ldexp(mm > 1.0 ? mm : 1.0, -23);
        double qd = clamped ? 0.0 : (fabs(Y[0] * dx + Y[1] * dy) + fabs(Y[1] * dx + Y[2] * dy)) * delta;
        if (rec && r.ncontrib < rec_cap) {
            contrib_t *e = &rec[r.ncontrib];
            e->li = i; e->alpha = alpha; e->T = T; e->G = G; e->sigma = sigma; e->dx = dx; e->dy = dy;
            e->clamped = clamped; e->amb_clamp = amb_clamp; e->delta = delta; e->qd = qd;
        }
        r.eT += alpha * qd / (1.0 - alpha);
        for (int ch = 0; ch < D; ch++) r.rgb[ch] += rgb[D * g + ch] * alpha * T;
        if (depth) r.dacc += depth[g] * alpha * T;
        T = nT;
        rT = rT_next;
        r.last_li = i;
        r.ncontrib++;
    }
    r.T = T;
    r.rT = rT;
    return r;
}

static int tile_selected(const uint8_t *tile_mask, int64_t c, int TX, int TY, int px, int py, int T)
{
    if (!tile_mask) return 1;
    return tile_mask[c * TX * TY + (py / T) * TX + (px / T)] != 0;
}

/* R1-R3 for every (selected) pixel.  out_last_gid = flat id c*N+n of the last
 * composited splat, -1 if none. Unselected pixels get rgb=bg, T=1, gid=-1. */
int or_render_fwd(const or_opts *o, int32_t C, int64_t N, int32_t W, int32_t H, const int32_t *radii,
                  const float *mean2d_f, const float *depth_f, const float *dec, const double *mean2d,
                  const double *conic,
                  const double *opac_eff, const double *rgb, const double *bg, const uint8_t *tile_mask,
                  double *out_rgb, double *out_alpha, double *out_T, int64_t *out_last_gid,
                  uint8_t *out_ambig, int32_t *out_ncontrib, const double *depth, double *out_depth,
                  const uint32_t *flips)
{
    int T = o->tile_size, TX = (W + T - 1) / T, TY = (H + T - 1) / T;
    const int D = n_channels(o);
    for (int64_t c = 0; c < C; c++) {
        camlist_t L;
        build_camlist(o, c, N, W, H, radii, mean2d_f, depth_f, &L);
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t pix = 0; pix < (int64_t)W * H; pix++) {
            int px = (int)(pix % W), py = (int)(pix / W);
            int64_t oi = c * W * H + pix;
            const double *b = bg ? bg + D * c : NULL;
            if (!tile_selected(tile_mask, c, TX, TY, px, py, T)) {
                for (int ch = 0; ch < D; ch++) out_rgb[D * oi + ch] = b ? b[ch] : 0.0;
                out_alpha[oi] = 0; out_T[oi] = 1; out_last_gid[oi] = -1;
                if (out_depth) out_depth[oi] = 0;
                if (out_ambig) out_ambig[oi] = 0;
                if (out_ncontrib) out_ncontrib[oi] = 0;
                continue;
            }
            pixres_t r = pixel_forward(o, &L, c, N, px, py, mean2d_f, dec, mean2d, conic, opac_eff, rgb, depth,
                                       NULL, 0, flips ? flips[oi] : 0u);
            for (int ch = 0; ch < D; ch++) out_rgb[D * oi + ch] = r.rgb[ch] + r.T * (b ? b[ch] : 0.0);  /* R3, Q25 */
            if (out_depth) out_depth[oi] = r.dacc;                                 /* no background term */
            out_alpha[oi] = 1.0 - r.T;
            out_T[oi] = r.T;
            out_last_gid[oi] = r.last_li >= 0 ? c * N + L.n[r.last_li] : -1;
            if (out_ambig) out_ambig[oi] = (uint8_t)(r.ambig < 255 ? r.ambig : 255);
            if (out_ncontrib) out_ncontrib[oi] = (int32_t)r.ncontrib;
        }
        free_camlist(&L);
    }
    return 0;
}

/* One pixel per query (camera cams[q], pixel (pxs[q], pys[q])) under the decision
 * outcomes flips[q] (see decide()): colour [D], T_final, the flat id of the last composited
 * splat (-1 if none) and the number of ambiguous decisions met.  Used to enumerate every
 * outcome an ambiguous pixel admits; the camera lists are built once per camera. */
int or_render_pixels(const or_opts *o, int32_t C, int64_t N, int32_t W, int32_t H, const int32_t *radii,
                     const float *mean2d_f, const float *depth_f, const float *dec, const double *mean2d,
                     const double *conic, const double *opac_eff, const double *rgb, const double *bg,
                     int64_t nq, const int32_t *cams, const int32_t *pxs, const int32_t *pys,
                     const uint32_t *flips, double *out_rgb, double *out_T, int64_t *out_last_gid,
                     int32_t *out_namb)
{
    const int D = n_channels(o);
    for (int64_t c = 0; c < C; c++) {
        int any = 0;
        for (int64_t q = 0; q < nq; q++) any |= cams[q] == c;
        if (!any) continue;
        camlist_t L;
        build_camlist(o, c, N, W, H, radii, mean2d_f, depth_f, &L);
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t q = 0; q < nq; q++) {
            if (cams[q] != c) continue;
            pixres_t r = pixel_forward(o, &L, c, N, pxs[q], pys[q], mean2d_f, dec, mean2d, conic, opac_eff, rgb,
                                       NULL, NULL, 0, flips[q]);
            const double *b = bg ? bg + D * c : NULL;
            for (int ch = 0; ch < D; ch++) out_rgb[D * q + ch] = r.rgb[ch] + r.T * (b ? b[ch] : 0.0);
            out_T[q] = r.T;
            out_last_gid[q] = r.last_li >= 0 ? c * N + L.n[r.last_li] : -1;
            out_namb[q] = r.ambig;
        }
        free_camlist(&L);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* B1-B6.  Per pixel: replay the forward to find the composited    */
/* sequence, then walk it back to front with the paper's recurrences           */
/* T_{n-1} = T_n/(1-alpha_{n-1}) and S.  Per-pixel terms are   */
/* written to per-pixel slots and summed serially in pixel order.              */
/* v2d layout per flat id g, 9 doubles:                                        */
/*   [0,1] v_mean2d  [2,3,4] v_conic (A,B,C)  [5,6,7] v_rgb  [8] v_opac_eff     */
/* a2d: same layout, sum over pixels of |term| with B4's v_alpha replaced by the */
/* sum of the magnitudes of its parts (the fp32 condition floor)    */
/* g_ambig[g] = 1 if g was evaluated at an ambiguous pixel.                     */
/* absg (optional) [C,N,2]: sum over pixels of |d L_pixel / d mu'| per axis (the  */
/* Absgrad statistic).                                                */
/* T_replay_err (optional) = max |T_replayed - T_forward| over all steps.      */
/* ------------------------------------------------------------------------- */
typedef struct { int32_t g; double v[10], va[10], vs[10], vd[9], rel; } term_t;   /* [9]: v_depth */

int or_render_bwd(const or_opts *o, int32_t C, int64_t N, int32_t W, int32_t H, const int32_t *radii,
                  const float *mean2d_f, const float *depth_f, const float *dec, const double *mean2d,
                  const double *conic,
                  const double *opac_eff, const double *rgb, const double *bg, const uint8_t *tile_mask,
                  const double *v_img, const double *v_alpha_img, double *v2d, double *a2d, double *s2d,
                  uint8_t *g_ambig, double *T_replay_err, const double *depth, const double *v_depth_img,
                  double *vz, double *az, double *sz, double *vfeat, double *absg, double *afeat,
                  const uint32_t *flips, int32_t *n2d, double *d2d, double *sfeat)
{
    int T = o->tile_size, TX = (W + T - 1) / T, TY = (H + T - 1) / T;
    const int D = n_channels(o);
    memset(v2d, 0, sizeof(double) * 9 * C * N);
    if (vfeat) memset(vfeat, 0, sizeof(double) * D * C * N);
    if (afeat) memset(afeat, 0, sizeof(double) * D * C * N);
    if (sfeat) memset(sfeat, 0, sizeof(double) * D * C * N);
    if (a2d) memset(a2d, 0, sizeof(double) * 9 * C * N);
    if (s2d) memset(s2d, 0, sizeof(double) * 9 * C * N);
    if (g_ambig) memset(g_ambig, 0, (size_t)C * N);
    if (vz) memset(vz, 0, sizeof(double) * C * N);
    if (az) memset(az, 0, sizeof(double) * C * N);
    if (sz) memset(sz, 0, sizeof(double) * C * N);
    if (absg) memset(absg, 0, sizeof(double) * 2 * C * N);
    if (n2d) memset(n2d, 0, sizeof(int32_t) * C * N);
    if (d2d) memset(d2d, 0, sizeof(double) * 9 * C * N);
    const int with_depth = depth && v_depth_img;
    double max_err = 0;
    for (int64_t c = 0; c < C; c++) {
        if (tile_mask) {   /* a camera without selected tiles contributes nothing */
            int any = 0;
            for (int64_t t = 0; t < (int64_t)TX * TY && !any; t++) any = tile_mask[c * TX * TY + t] != 0;
            if (!any) continue;
        }
        camlist_t L;
        build_camlist(o, c, N, W, H, radii, mean2d_f, depth_f, &L);
        int64_t P = (int64_t)W * H;
        int32_t *cnt = (int32_t *)calloc(P, sizeof(int32_t));
        /* pass 1: composited count per pixel */
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t pix = 0; pix < P; pix++) {
            int px = (int)(pix % W), py = (int)(pix / W);
            if (!tile_selected(tile_mask, c, TX, TY, px, py, T)) continue;
            pixres_t r = pixel_forward(o, &L, c, N, px, py, mean2d_f, dec, mean2d, conic, opac_eff, rgb, NULL,
                                       NULL, 0, flips ? flips[c * P + pix] : 0u);
            cnt[pix] = (int32_t)r.ncontrib;
            if (r.ambig && g_ambig) {
                /* mark every splat this pixel evaluated (in-tile, up to termination) */
                int tx = px / T, ty = py / T;
                for (int64_t i = 0; i < r.end_li; i++) {
                    const int32_t *rc = &L.rect[4 * i];
                    if (tx < rc[0] || tx >= rc[1] || ty < rc[2] || ty >= rc[3]) continue;
                    int64_t g = c * N + L.n[i];
#pragma omp atomic write
                    g_ambig[g] = 1;
                }
            }
        }
        int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (P + 1));
        off[0] = 0;
        for (int64_t pix = 0; pix < P; pix++) off[pix + 1] = off[pix] + cnt[pix];
        int64_t tot = off[P];
        term_t *terms = (term_t *)malloc(sizeof(term_t) * (tot > 0 ? tot : 1));
        /* per-term feature gradients (N-D mode: D values per term; RGB mode uses v[5..7]) */
        double *tvf = vfeat ? (double *)malloc(sizeof(double) * D * (tot > 0 ? tot : 1)) : NULL;
        double *errs = (double *)calloc(P, sizeof(double));
        /* pass 2: per-pixel backward */
#pragma omp parallel
        {
            int64_t cap = 1024;
            contrib_t *rec = (contrib_t *)malloc(sizeof(contrib_t) * cap);
#pragma omp for schedule(dynamic, 64)
            for (int64_t pix = 0; pix < P; pix++) {
                if (cnt[pix] == 0) continue;
                int px = (int)(pix % W), py = (int)(pix / W);
                if (cnt[pix] > cap) {
                    cap = cnt[pix];
                    rec = (contrib_t *)realloc(rec, sizeof(contrib_t) * cap);
                }
                pixres_t r = pixel_forward(o, &L, c, N, px, py, mean2d_f, dec, mean2d, conic, opac_eff, rgb, NULL,
                                           rec, cap, flips ? flips[c * P + pix] : 0u);
                int64_t oi = c * P + pix;
                const double *vC = &v_img[D * oi];
                double vA = v_alpha_img ? v_alpha_img[oi] : 0.0;
                const double *b = bg ? bg + D * c : NULL;
                double bgdot = 0.0;
                if (b)
                    for (int ch = 0; ch < D; ch++) bgdot += b[ch] * vC[ch];
                double Tfin = r.T;
                double vD = with_depth ? v_depth_img[oi] : 0.0;   /* d L / d (accumulated depth) */
                double Tn = Tfin;                /* B1 */
                double S[OR_MAX_CH] = {0}, Sd = 0;  /* Sd: the depth channel's S */
                double err = 0;
                for (int64_t k = r.ncontrib - 1; k >= 0; k--) {
                    const contrib_t *e = &rec[k];
                    int64_t g = c * N + L.n[e->li];
                    double alpha = e->alpha;
                    double ra = 1.0 / (1.0 - alpha);
                    Tn = Tn * ra;                /* B2: T_{n-1} = T_n / (1 - alpha_{n-1}) */
                    double d = fabs(Tn - e->T);
                    if (d > err) err = d;
                    double fac = alpha * Tn;
                    term_t *tm = &terms[off[pix] + k];
                    tm->g = (int32_t)g;
                    for (int ch = 0; ch < 3; ch++) tm->v[5 + ch] = D == 3 ? fac * vC[ch] : 0.0;  /* B3 */
                    for (int ch = 0; ch < 3; ch++) tm->va[5 + ch] = fabs(tm->v[5 + ch]);
                    if (tvf)
                        for (int ch = 0; ch < D; ch++) tvf[(off[pix] + k) * D + ch] = fac * vC[ch];
                    double z = with_depth ? depth[g] : 0.0;
                    tm->v[9] = fac * vD;                                           /* depth as a channel: B3 */
                    tm->va[9] = fabs(tm->v[9]);
                    double v_alpha = 0;                                            /* B4 */
                    for (int ch = 0; ch < D; ch++) v_alpha += (rgb[D * g + ch] * Tn - S[ch] * ra) * vC[ch];
                    v_alpha += (z * Tn - Sd * ra) * vD;                            /* depth channel */
                    v_alpha += -Tfin * ra * bgdot + Tfin * ra * vA;
                    /* magnitude of B4 before its internal cancellation (c T vs S/(1-alpha)):
                     * the condition floor a2d of the v_alpha-dependent gradients uses it */
                    double v_alpha_abs = fabs(Tfin * ra * bgdot) + fabs(Tfin * ra * vA);
                    for (int ch = 0; ch < D; ch++)
                        v_alpha_abs += fabs(rgb[D * g + ch] * Tn * vC[ch]) + fabs(S[ch] * ra * vC[ch]);
                    v_alpha_abs += fabs(z * Tn * vD) + fabs(Sd * ra * vD);

                    for (int ch = 0; ch < D; ch++) S[ch] += rgb[D * g + ch] * fac;  /* B5 */
                    Sd += z * fac;
                    /* tolerance model: an ambiguous alpha_max decision (Q13/Q24) admits both B6
                     * outcomes, clamped (no sigma / opacity gradient) and not; vd = the
                     * magnitude of the difference, i.e. of the unclamped B6 terms */
                    for (int j = 0; j < 9; j++) tm->vd[j] = 0;
                    if (e->amb_clamp) {
                        double vs_ = opac_eff[g] * e->G * fabs(v_alpha);
                        const double *Y = &conic[3 * g];
                        tm->vd[8] = e->G * fabs(v_alpha);
                        tm->vd[2] = vs_ * 0.5 * e->dx * e->dx;
                        tm->vd[3] = vs_ * fabs(e->dx * e->dy);
                        tm->vd[4] = vs_ * 0.5 * e->dy * e->dy;
                        tm->vd[0] = vs_ * fabs(Y[0] * e->dx + Y[1] * e->dy);
                        tm->vd[1] = vs_ * fabs(Y[1] * e->dx + Y[2] * e->dy);
                    }
                    if (!e->clamped) {                                           /* B6 (Q24) */
                        tm->v[8] = e->G * v_alpha;
                        double v_sigma = -opac_eff[g] * e->G * v_alpha;
                        const double *Y = &conic[3 * g];
                        tm->v[2] = v_sigma * 0.5 * e->dx * e->dx;
                        tm->v[3] = v_sigma * e->dx * e->dy;
                        tm->v[4] = v_sigma * 0.5 * e->dy * e->dy;
                        tm->v[0] = v_sigma * (Y[0] * e->dx + Y[1] * e->dy);
                        tm->v[1] = v_sigma * (Y[1] * e->dx + Y[2] * e->dy);
                        double vsa = opac_eff[g] * e->G * v_alpha_abs;
                        tm->va[8] = e->G * v_alpha_abs;
                        tm->va[2] = vsa * 0.5 * e->dx * e->dx;
                        tm->va[3] = vsa * fabs(e->dx * e->dy);
                        tm->va[4] = vsa * 0.5 * e->dy * e->dy;
                        tm->va[0] = vsa * (fabs(Y[0] * e->dx) + fabs(Y[1] * e->dy));
                        tm->va[1] = vsa * (fabs(Y[1] * e->dx) + fabs(Y[2] * e->dy));
                        /* first-order effect of the fp32 rounding of mu' (delta, 1 ulp) on the
                         * polynomial factors of B6 */
                        tm->vs[2] = vsa * fabs(e->dx) * e->delta;
                        tm->vs[3] = vsa * (fabs(e->dx) + fabs(e->dy)) * e->delta;
                        tm->vs[4] = vsa * fabs(e->dy) * e->delta;
                        tm->vs[0] = vsa * (fabs(Y[0]) + fabs(Y[1])) * e->delta;
                        tm->vs[1] = vsa * (fabs(Y[1]) + fabs(Y[2])) * e->delta;
                    } else {
                        tm->v[8] = tm->v[0] = tm->v[1] = tm->v[2] = tm->v[3] = tm->v[4] = 0;
                        tm->va[8] = tm->va[0] = tm->va[1] = tm->va[2] = tm->va[3] = tm->va[4] = 0;
                        tm->vs[0] = tm->vs[1] = tm->vs[2] = tm->vs[3] = tm->vs[4] = 0;
                    }
                    /* ... and through alpha (this splat's qd, all splats' via T and S) */
                    for (int j = 0; j < 10; j++) {
                        if (j >= 5) tm->vs[j] = 0;   /* rgb, opacity, depth: only the alpha path */
                        /* + the fp32 rounding of the T recurrence (1 - alpha amplifies it near
                         * alpha_max): every T the kernel forms, forward or recovered backward
                         * from T_final, is within the pixel's r_T of the exact one */
                        tm->vs[j] += tm->va[j] * (e->qd + r.eT + r.rT);
                    }
                    tm->rel = e->qd + r.eT + r.rT;
                }
                errs[pix] = err;
            }
            free(rec);
        }
        /* pass 3: serial reduction in pixel order */
        for (int64_t i = 0; i < tot; i++) {
            int32_t g = terms[i].g;
            for (int j = 0; j < 9; j++) {
                v2d[9 * (int64_t)g + j] += terms[i].v[j];
                if (a2d) a2d[9 * (int64_t)g + j] += terms[i].va[j];
                if (s2d) s2d[9 * (int64_t)g + j] += terms[i].vs[j];
            }
            if (vz) vz[g] += terms[i].v[9];
            if (n2d) n2d[g] += 1;   /* tolerance model: terms summed into g (atomic-order bound) */
            if (d2d)
                for (int j = 0; j < 9; j++) d2d[9 * (int64_t)g + j] += terms[i].vd[j];
            /* Absgrad (App. Absgrad): per-pixel absolute view-space gradients */
            if (absg) {
                absg[2 * (int64_t)g + 0] += fabs(terms[i].v[0]);
                absg[2 * (int64_t)g + 1] += fabs(terms[i].v[1]);
            }
            if (tvf)
                for (int ch = 0; ch < D; ch++) vfeat[(int64_t)g * D + ch] += tvf[i * D + ch];
            if (tvf && afeat)   /* tolerance model: sum over pixels of |fac v_C| per channel */
                for (int ch = 0; ch < D; ch++) afeat[(int64_t)g * D + ch] += fabs(tvf[i * D + ch]);
            if (tvf && sfeat)   /* ... times the relative sensitivity of fac = alpha T (as vs for rgb) */
                for (int ch = 0; ch < D; ch++) sfeat[(int64_t)g * D + ch] += fabs(tvf[i * D + ch]) * terms[i].rel;
            if (az) az[g] += terms[i].va[9];
            if (sz) sz[g] += terms[i].vs[9];
        }
        for (int64_t pix = 0; pix < P; pix++)
            if (errs[pix] > max_err) max_err = errs[pix];
        free(errs); free(terms); free(tvf); free(off); free(cnt);
        free_camlist(&L);
    }
    if (T_replay_err) *T_replay_err = max_err;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* P1-P9: projection backward, summed over cameras (Q30).          */
/* v2d is the 9-double layout of or_render_bwd.  Outputs fully overwritten:    */
/* v_means [N,3], v_quats [N,4], v_scales [N,3], v_opac [N],                   */
/* v_colors [N,K,3] (SH) or [N,3] (direct).                                    */
/* ------------------------------------------------------------------------- */
int or_project_bwd(const or_opts *o, int64_t N, int32_t C, int32_t W, int32_t H, const float *means,
                   const float *quats, const float *scales, const float *opacities, const float *colors,
                   int32_t K, const float *viewmats, const float *Ks, const int32_t *radii, const double *v2d,
                   double *v_means, double *v_quats, double *v_scales, double *v_opac, double *v_colors,
                   const double *vz, double *v_viewmats, int32_t absmode)
{
    /* absmode (tolerance model, not a result): the same chain with every operand replaced by
     * its magnitude and every subtraction by an addition, i.e. |Jacobian| applied to the
     * (non-negative) inputs v2d, vz -- the running bound sum |terms| of each output, used to
     * propagate per-element error bounds of the 2D gradients to the parameter gradients and
     * to size the fp32 rounding floor of the projection backward (DESIGN.md parity contract). */
    const double sg = absmode ? 1.0 : -1.0;     /* sign of every subtracted term */
#define AV(x) (absmode ? fabs(x) : (x))
    int64_t stride = o->sh_degree >= 0 ? (int64_t)K * 3 : 3;
    /* pose gradients (App. pose optimisation): per-thread partial sums
     * over Gaussians, summed in thread order after the loop */
    int nthr = 1;
#ifdef _OPENMP
    nthr = omp_get_max_threads();
#endif
    double *vpart = v_viewmats ? (double *)calloc((size_t)nthr * C * 16, sizeof(double)) : NULL;
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
        double gm[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gs[3] = {0, 0, 0}, go = 0;
        double *gc = &v_colors[stride * n];
        for (int64_t j = 0; j < stride; j++) gc[j] = 0;
        for (int64_t c = 0; c < C; c++) {
            int64_t idx = c * N + n;
            if (radii[2 * idx] <= 0 || radii[2 * idx + 1] <= 0) continue;
            double vg[9];
            for (int j = 0; j < 9; j++) vg[j] = AV(v2d[9 * idx + j]);
            if (absmode == 2)   /* only the colour channels (the SH clamp alternative below) */
                vg[0] = vg[1] = vg[2] = vg[3] = vg[4] = vg[8] = 0;
            proj64_t P;
            project64(o, W, H, means + 3 * n, quats + 4 * n, scales + 3 * n, opacities[n],
                      colors + stride * n, K, viewmats + 16 * c, Ks + 9 * c, &P);
            if (absmode) abs_proj(&P);
            /* P1: o_eff = o * comp */
            go += vg[8] * P.comp;
            double v_comp = vg[8] * P.o;
            /* P2: Y = Spb^-1, G_Y = [[vA, vB/2],[vB/2, vC]], v_Spb = -Y G_Y Y */
            double Y[2][2] = {{P.conic[0], P.conic[1]}, {P.conic[1], P.conic[2]}};
            double GY[2][2] = {{vg[2], 0.5 * vg[3]}, {0.5 * vg[3], vg[4]}};
            double YG[2][2], vSp[2][2];
            for (int i = 0; i < 2; i++)
                for (int j = 0; j < 2; j++) YG[i][j] = Y[i][0] * GY[0][j] + Y[i][1] * GY[1][j];
            for (int i = 0; i < 2; i++)
                for (int j = 0; j < 2; j++) vSp[i][j] = sg * (YG[i][0] * Y[0][j] + YG[i][1] * Y[1][j]);
            /* P3 (AA only): d comp / d Sigma' = comp/2 (Sigma'^-1 - Spb^-1) (derived from P:281) */
            if (o->antialiased && P.det > 0) {
                double Si[2][2] = {{P.Sp[1][1] / P.det, sg * P.Sp[0][1] / P.det},
                                   {sg * P.Sp[1][0] / P.det, P.Sp[0][0] / P.det}};
                for (int i = 0; i < 2; i++)
                    for (int j = 0; j < 2; j++) vSp[i][j] += v_comp * 0.5 * P.comp * (Si[i][j] + sg * Y[i][j]);
            }
            /* P4: v_Sc = J^T vSp J; v_J = vSp J Sc^T + vSp^T J Sc (Q11) */
            double vSc[3][3], vJ[2][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0;
                    for (int k = 0; k < 2; k++)
                        for (int l = 0; l < 2; l++) acc += P.J[k][i] * vSp[k][l] * P.J[l][j];
                    vSc[i][j] = acc;
                }
            for (int i = 0; i < 2; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0;
                    for (int k = 0; k < 2; k++)
                        for (int l = 0; l < 3; l++)
                            acc += vSp[i][k] * P.J[k][l] * P.Sc[j][l] + vSp[k][i] * P.J[k][l] * P.Sc[l][j];
                    vJ[i][j] = acc;
                }
            /* P5: v_t through J (exact derivative with the clamp of Q27)
             * and through mu' (re-derived from P:790-791, Q10) */
            double tx = P.t[0], ty = P.t[1], tz = P.t[2];
            double fx = P.fx, fy = P.fy, tz2 = tz * tz, tz3 = tz2 * tz;
            double vt[3] = {0, 0, 0};
            vt[2] += sg * fx / tz2 * vJ[0][0] + sg * fy / tz2 * vJ[1][1];
            if (!P.clamp_x) {
                vt[0] += sg * fx / tz2 * vJ[0][2];
                vt[2] += 2.0 * fx * tx / tz3 * vJ[0][2];
            } else {
                vt[2] += fx * P.txc / tz3 * vJ[0][2];
            }
            if (!P.clamp_y) {
                vt[1] += sg * fy / tz2 * vJ[1][2];
                vt[2] += 2.0 * fy * ty / tz3 * vJ[1][2];
            } else {
                vt[2] += fy * P.tyc / tz3 * vJ[1][2];
            }
            vt[0] += fx / tz * vg[0];
            vt[1] += fy / tz * vg[1];
            vt[2] += sg * (fx * tx / tz2) * vg[0] + sg * (fy * ty / tz2) * vg[1];
            if (vz) vt[2] += AV(vz[idx]);                  /* depth = t_z (F4; depth rendering P:250) */
            double *vW = vpart ? vpart + ((size_t)tid * C + c) * 16 : NULL;
            if (vW) {
                /* t = W mu + w: dL/dW += v_t mu^T, dL/dw += v_t */
                for (int i = 0; i < 3; i++) {
                    for (int j = 0; j < 3; j++) vW[4 * i + j] += vt[i] * P.mu[j];
                    vW[4 * i + 3] += vt[i];
                }
                /* Sigma_c = W Sigma W^T (Fig. P:423): dL/dW += (vSc + vSc^T) W Sigma */
                for (int i = 0; i < 3; i++)
                    for (int j = 0; j < 3; j++) {
                        double acc = 0;
                        for (int k = 0; k < 3; k++)
                            for (int l = 0; l < 3; l++) acc += (vSc[i][k] + vSc[k][i]) * P.Wr[k][l] * P.Sig[l][j];
                        vW[4 * i + j] += acc;
                    }
            }
            /* P6: v_mu += W^T v_t, v_Sigma = W^T v_Sc W */
            for (int i = 0; i < 3; i++)
                for (int k = 0; k < 3; k++) gm[i] += P.Wr[k][i] * vt[k];
            double vS[3][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0;
                    for (int k = 0; k < 3; k++)
                        for (int l = 0; l < 3; l++) acc += P.Wr[k][i] * vSc[k][l] * P.Wr[l][j];
                    vS[i][j] = acc;
                }
            /* P7: colour */
            const double *vrgb = &vg[5];
            if (o->sh_degree >= 0) {
                int deg = o->sh_degree, nb = (deg + 1) * (deg + 1);
                double Yb[16], dY[16][3];
                if (absmode) {
                    sh_basis_mag(deg, P.dir[0], P.dir[1], P.dir[2], Yb, dY);
                } else {
                    sh_basis(deg, P.dir[0], P.dir[1], P.dir[2], Yb);
                    sh_basis_grad(deg, P.dir[0], P.dir[1], P.dir[2], dY);
                }
                double vraw[3];
                for (int ch = 0; ch < 3; ch++) {
                    int on = P.raw[ch] > 0;   /* colour = max(0, raw): no gradient where clamped (Q22) */
                    /* absmode 2 (tolerance model): the channels whose clamp decision lies within
                     * the fp32 rounding of raw (64 u of its term magnitudes) admit both outcomes;
                     * the bound of the alternative is the full magnitude of their path */
                    if (absmode == 2) on = fabs(P.raw[ch]) <= 64 * OR_U * P.rawabs[ch];
                    vraw[ch] = on ? vrgb[ch] : 0.0;
                }
                double vdir[3] = {0, 0, 0};
                for (int j = 0; j < nb; j++) {
                    double shv = 0;
                    for (int ch = 0; ch < 3; ch++) {
                        gc[3 * j + ch] += AV(Yb[j]) * vraw[ch];
                        shv += AV((double)colors[stride * n + 3 * j + ch]) * vraw[ch];
                    }
                    for (int d = 0; d < 3; d++) vdir[d] += AV(dY[j][d]) * shv;
                }
                /* dir = e/|e|, d dir/d mu = (I - dir dir^T)/|e| */
                double dd = P.dir[0] * vdir[0] + P.dir[1] * vdir[1] + P.dir[2] * vdir[2];
                double ve[3];
                for (int i = 0; i < 3; i++) ve[i] = (vdir[i] + sg * P.dir[i] * dd) / P.enorm;
                for (int i = 0; i < 3; i++) gm[i] += ve[i];
                /* e = mu - campos, campos = -W^T w: dL/dW_ki += ve_i w_k, dL/dw_k += (W ve)_k */
                double *vW = vpart ? vpart + ((size_t)tid * C + c) * 16 : NULL;
                if (vW)
                    for (int k = 0; k < 3; k++)
                        for (int i = 0; i < 3; i++) {
                            vW[4 * k + i] += ve[i] * P.w[k];
                            vW[4 * k + 3] += P.Wr[k][i] * ve[i];
                        }
            } else if (absmode != 2) {   /* direct colours: no clamp, no alternative */
                for (int ch = 0; ch < 3; ch++) gc[ch] += vrgb[ch];
            }
            /* P8: Sigma = M M^T -> v_M = (vS + vS^T) M; M = R S -> v_R = v_M S, v_s */
            double vM[3][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0;
                    for (int k = 0; k < 3; k++) acc += (vS[i][k] + vS[k][i]) * P.M[k][j];
                    vM[i][j] = acc;
                }
            for (int j = 0; j < 3; j++) {
                double acc = 0;
                for (int i = 0; i < 3; i++) acc += P.R[i][j] * vM[i][j];
                gs[j] += acc;
            }
            double vR[3][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) vR[i][j] = vM[i][j] * P.s[j];
            /* P9: dR/d(w,x,y,z) at q_hat, then the normalisation */
            double w = P.qh[0], x = P.qh[1], y = P.qh[2], z = P.qh[3];
            double dRw[3][3] = {{0, sg * z, y}, {z, 0, sg * x}, {sg * y, x, 0}};
            double dRx[3][3] = {{0, y, z}, {y, sg * 2 * x, sg * w}, {z, w, sg * 2 * x}};
            double dRy[3][3] = {{sg * 2 * y, x, w}, {x, 0, z}, {sg * w, z, sg * 2 * y}};
            double dRz[3][3] = {{sg * 2 * z, sg * w, x}, {w, sg * 2 * z, y}, {x, y, 0}};
            double vqh[4] = {0, 0, 0, 0};
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    vqh[0] += 2.0 * dRw[i][j] * vR[i][j];
                    vqh[1] += 2.0 * dRx[i][j] * vR[i][j];
                    vqh[2] += 2.0 * dRy[i][j] * vR[i][j];
                    vqh[3] += 2.0 * dRz[i][j] * vR[i][j];
                }
            double dot = vqh[0] * P.qh[0] + vqh[1] * P.qh[1] + vqh[2] * P.qh[2] + vqh[3] * P.qh[3];
            for (int i = 0; i < 4; i++) gq[i] += (vqh[i] + sg * dot * P.qh[i]) / P.qn;
        }
        for (int i = 0; i < 3; i++) v_means[3 * n + i] = gm[i], v_scales[3 * n + i] = gs[i];
        for (int i = 0; i < 4; i++) v_quats[4 * n + i] = gq[i];
        v_opac[n] = go;
    }
    if (v_viewmats) {
        memset(v_viewmats, 0, sizeof(double) * 16 * C);
        for (int t = 0; t < nthr; t++)
            for (int64_t k = 0; k < 16 * (int64_t)C; k++) v_viewmats[k] += vpart[(size_t)t * C * 16 + k];
        free(vpart);
    }
#undef AV
    return 0;
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_num_threads(int n)
{
#ifdef _OPENMP
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}
