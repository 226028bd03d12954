/*
 * oracle/port/ccport.c — TEST INFRASTRUCTURE ONLY (a checker, never shipped).
 *
 * A plain-C11 restatement of the reference's encode iteration, written per
 * latent / per pixel (no batching, no vectorisation tricks), behind the same C
 * ABI as the B200 library (include/coolchic_b200.h).  Every routine cites the
 * reference file:line it restates (paths relative to
 * /root/reference/proj/include/coolcodec).  Arithmetic is fp32 with fp64
 * accumulators exactly where the reference uses them; the initialisers use
 * fmaf where the reference build contracts (-ffp-contract=fast), so
 * fresh_candidate is bit-exact.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "coolchic_b200.h"
#include "coolchic_synth.h"

#define MAXG 16
#define MAXT 64
#define MAXCTX 144
#define NSLOT 8
#define NCAND 16

static _Thread_local char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

/* ------------------------------------------------ mathutil.hpp:18-103 --- */
static uint64_t splitmix64(uint64_t z) { return ccs_splitmix64(z); }
static uint64_t hash_combine(uint64_t a, uint64_t b) { return ccs_hash_combine(a, b); }
static float counter_gauss(uint64_t stream, uint64_t index) {  /* :35-40 */
    const uint64_t h = splitmix64(stream + index);
    const double u1 = ((double)(h >> 40) + 1.0) * 0x1.0p-24;
    const double u2 = (double)((h >> 16) & 0xffffffu) * 0x1.0p-24;
    return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}
static float counter_uniform(uint64_t stream, uint64_t index, float lo, float hi) { /* :42-44 */
    return fmaf(hi - lo, (float)ccs_unit(splitmix64(stream + index)), lo);
}
static float fminr(float a, float b) { return (b < a) ? b : a; } /* std::min(a,b) */
static float fmaxr(float a, float b) { return (a < b) ? b : a; } /* std::max(a,b) */
static float cc_exp(float x) { /* :55-71 */
    x = fminr(88.0f, fmaxr(-87.0f, x));
    /* the reference build (-ffp-contract=fast) fuses both uses of x*log2(e) */
    const float nf = floorf(fmaf(x, 1.44269504088896341f, 0.5f));
    const float t = fmaf(x, 1.44269504088896341f, -nf) * 0.69314718055994531f;
    float p = 0.0013888889f;
    p = fmaf(t, p, 0.008333334f);
    p = fmaf(t, p, 0.041666668f);
    p = fmaf(t, p, 0.16666667f);
    p = fmaf(t, p, 0.5f);
    p = fmaf(t, p, 1.0f);
    p = fmaf(t, p, 1.0f);
    union { uint32_t u; float f; } s;
    s.u = (uint32_t)((int32_t)nf + 127) << 23;
    return p * s.f;
}
static float cc_log(float x) { /* :73-86 */
    union { float f; uint32_t u; } b;
    b.f = x;
    int e = (int)(b.u >> 23) - 127;
    union { uint32_t u; float f; } m;
    m.u = (b.u & 0x007fffffu) | 0x3f800000u;
    float mm = m.f;
    if (mm > 1.41421356f) { mm *= 0.5f; ++e; }
    const float s = (mm - 1.0f) / (mm + 1.0f);
    const float s2 = s * s;
    float p = 0.11111111f;
    p = fmaf(s2, p, 0.14285715f);
    p = fmaf(s2, p, 0.2f);
    p = fmaf(s2, p, 0.33333333f);
    p = fmaf(s2, p, 1.0f);
    return fmaf(2.0f * s, p, (float)e * 0.69314718f);
}
static float cc_tanh(float x) { /* :88-94 */
    float ax = fabsf(x);
    ax = fminr(ax, 9.0f);
    const float t = cc_exp(-2.0f * ax);
    const float r = (1.0f - t) / (1.0f + t);
    return x < 0.0f ? -r : r;
}
/* layers.hpp:546-577 */
static float softround_denom(float temp) { return 2.0f * cc_tanh(1.0f / (2.0f * temp)); }
static float softround_value(float x, float temp) {
    const float f = floorf(x);
    const float d = x - f - 0.5f;
    return f + 0.5f + cc_tanh(d / temp) / softround_denom(temp);
}
/* layers.hpp:591-609 */
#define SIGMA_MIN 0.06f
#define SIGMA_MAX 256.0f
#define PFLOOR (1.0f / 65536.0f)
#define INV_SQRT2 0.7071067811865476f
static float laplace_bits(float v, float mu, float sigma) {
    const float b = sigma * INV_SQRT2;
    const float u = fabsf(v - mu);
    const float e1 = cc_exp(-(u + 0.5f) / b);
    const float e2 = cc_exp(-fabsf(u - 0.5f) / b);
    const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
    return -(cc_log(fmaxr(p, PFLOOR)) * 1.4426950408889634f);
}
/* latent.hpp:86-91 */
static int32_t quantize_value(float y, int amp) {
    long q = lroundf(y);
    if (q > amp) q = amp;
    if (q < -amp) q = -amp;
    return (int32_t)q;
}

/* ------------------------------------------------------------ trainer --- */
typedef struct {
    int level, hyper, rows, cols, slot, rdim;
    int64_t off;   /* flat latent offset */
} Grid;

typedef struct {
    char name[32];
    int rows, cols, size, off;
} Tensor;

typedef struct {
    int valid;
    double cost;
    float *y, *p;
} Snap;

typedef struct {
    int valid;
    double cost;
    float *y, *m, *v, *p, *nm, *nv;
    int64_t lat_t[MAXG], nn_t[MAXT];
} Cand;

struct cc_trainer {
    int H, W, L, hyper, n_grids, P, S, F, D, Wd, synF, posts, stab, use_hyper;
    int64_t npix, n_lat;
    int ctx_dy[MAXCTX], ctx_dx[MAXCTX];
    Grid g[MAXG];
    int main_gi[8];
    int n_slots, slot_gi[3];
    /* parameter layout (model.hpp:158-171) */
    int n_t, n_par;
    Tensor t[MAXT];
    int o_l1w, o_l1b, o_l2w, o_l2b, o_hw, o_hb, o_astab, o_ifw[3], o_ifb[3], o_tc[8], o_rf[8];
    int o_c1w, o_c1b, o_c2w, o_c2b, o_pw[2], o_pb[2], o_sstab;
    cc_encoder_config enc;
    char log_path[512];
    /* state */
    int loaded;
    float *img, *y, *yg, *lm, *lv, *par, *grad, *nm, *nv, *th1, *th2;
    int32_t* q;
    int64_t lat_t[MAXG], nn_t[MAXT];
    float* pv[MAXG];   /* padded values */
    float* pg[MAXG];   /* padded grads */
    int stride[MAXG];
    float *z, *dz, *h1, *trunk, *post[2], *xhat, *dx;
    float* ups_row[8][8]; /* [k][j] caches */
    float* ups_col[8][8];
    float* ups_out[8][8];
    double last_mse, last_bits, cur_cost;
    int64_t global_iter;
    int skipped;
    Snap snaps[NSLOT];
    Cand cands[NCAND];
    double* records;
    int n_records;
};

static int cdiv(int a, int b) { return (a + b - 1) / b; }

static float* zalloc(size_t n) {
    float* p = (float*)calloc(n ? n : 1, sizeof(float));
    if (!p) { fprintf(stderr, "ccport: out of memory\n"); abort(); }
    return p;
}

/* make_context_offsets (entropy_model.hpp:24-45) */
typedef struct { int d2, dy, dx; } CtxCand;
static int ctx_cmp(const void* a, const void* b) {
    const CtxCand* x = (const CtxCand*)a;
    const CtxCand* y = (const CtxCand*)b;
    if (x->d2 != y->d2) return x->d2 < y->d2 ? -1 : 1;
    if (x->dy != y->dy) return x->dy < y->dy ? -1 : 1;
    return x->dx < y->dx ? -1 : (x->dx > y->dx);
}

static int add_tensor(cc_trainer* T, const char* name, int rows, int cols) {
    Tensor* t = &T->t[T->n_t++];
    snprintf(t->name, sizeof(t->name), "%s", name);
    t->rows = rows;
    t->cols = cols;
    t->size = rows * cols;
    t->off = T->n_par;
    T->n_par += t->size;
    return t->off;
}

static int build(cc_trainer* T, const cc_decoder_config* dec) {
    T->L = (int64_t)T->H * T->W < 1000000 ? 7 : 8;  /* config.hpp:84 */
    T->use_hyper = dec->use_hyperlatents;
    T->hyper = dec->use_hyperlatents ? T->L - 4 : 0;
    T->S = dec->spatial_ctx;
    T->F = dec->ifce_dim;
    T->D = T->S + T->F;
    T->Wd = dec->arm_width;
    T->synF = dec->synth_hidden;
    T->posts = dec->synth_posts;
    T->stab = dec->use_stabilizer;
    if (T->posts < 0 || T->posts > 2) return fail(CC_ERR_CONFIG, "synth_posts must be <= 2");
    CtxCand c[8 * 17 + 8];
    int nc = 0;
    for (int dy = -8; dy <= 0; ++dy)
        for (int dx = -8; dx <= 8; ++dx) {
            if (dy == 0 && dx >= 0) continue;
            c[nc].d2 = dy * dy + dx * dx;
            c[nc].dy = dy;
            c[nc].dx = dx;
            ++nc;
        }
    qsort(c, (size_t)nc, sizeof(CtxCand), ctx_cmp);
    if (T->S > nc) return fail(CC_ERR_CONFIG, "spatial context too large");
    int pad = 0;
    for (int i = 0; i < T->S; ++i) {
        T->ctx_dy[i] = c[i].dy;
        T->ctx_dx[i] = c[i].dx;
        if (-c[i].dy > pad) pad = -c[i].dy;
        if (abs(c[i].dx) > pad) pad = abs(c[i].dx);
    }
    T->P = pad > 1 ? pad : 1;
    /* build_latents (latent.hpp:46-70) */
    int n = 0;
    int64_t off = 0;
    if (T->use_hyper)
        for (int k = T->L - 1; k >= 4; --k) {
            T->g[n].level = k;
            T->g[n].hyper = 1;
            ++n;
        }
    for (int k = T->L - 1; k >= 0; --k) {
        T->g[n].level = k;
        T->g[n].hyper = 0;
        T->main_gi[k] = n;
        ++n;
    }
    T->n_grids = n;
    for (int i = 0; i < n; ++i) {
        Grid* g = &T->g[i];
        g->rows = cdiv(T->H, 1 << g->level);
        g->cols = cdiv(T->W, 1 << g->level);
        g->off = off;
        off += (int64_t)g->rows * g->cols;
        g->slot = -1;
        g->rdim = 0;
    }
    T->n_lat = off;
    T->n_slots = 0;
    if (T->F > 0)
        for (int k = 0; k < 3 && k < T->L; ++k) {
            const int gi = T->main_gi[k];
            T->g[gi].slot = T->n_slots;
            T->g[gi].rdim = T->hyper + T->L - 1 - k;  /* model.hpp:70-71 */
            T->slot_gi[T->n_slots++] = gi;
        }
    /* make_model (model.hpp:80-123) + for_each_param order */
    char nm[32];
    T->o_l1w = add_tensor(T, "arm.l1.w", T->Wd, T->D);
    T->o_l1b = add_tensor(T, "arm.l1.b", 1, T->Wd);
    T->o_l2w = add_tensor(T, "arm.l2.w", T->Wd, T->Wd);
    T->o_l2b = add_tensor(T, "arm.l2.b", 1, T->Wd);
    T->o_hw = add_tensor(T, "arm.head.w", 2, T->Wd);
    T->o_hb = add_tensor(T, "arm.head.b", 1, 2);
    T->o_astab = T->stab ? add_tensor(T, "arm.stab", 2, T->D) : -1;
    for (int s = 0; s < T->n_slots; ++s) {
        const int rd = T->g[T->slot_gi[s]].rdim;
        snprintf(nm, sizeof(nm), "ifce%d.w", s);
        T->o_ifw[s] = add_tensor(T, nm, T->F, rd);
        snprintf(nm, sizeof(nm), "ifce%d.b", s);
        T->o_ifb[s] = add_tensor(T, nm, 1, T->F);
    }
    for (int j = 0; j < T->L - 1; ++j) {
        snprintf(nm, sizeof(nm), "ups%d.tconv", j);
        T->o_tc[j] = add_tensor(T, nm, 1, 4);
        snprintf(nm, sizeof(nm), "ups%d.refine", j);
        T->o_rf[j] = add_tensor(T, nm, 1, 3);
    }
    T->o_c1w = add_tensor(T, "syn.c1.w", T->synF, T->L);
    T->o_c1b = add_tensor(T, "syn.c1.b", 1, T->synF);
    T->o_c2w = add_tensor(T, "syn.c2.w", 3, T->synF);
    T->o_c2b = add_tensor(T, "syn.c2.b", 1, 3);
    for (int i = 0; i < T->posts; ++i) {
        snprintf(nm, sizeof(nm), "syn.post%d.w", i);
        T->o_pw[i] = add_tensor(T, nm, 3, 27);
    }
    for (int i = 0; i < T->posts; ++i) {
        snprintf(nm, sizeof(nm), "syn.post%d.b", i);
        T->o_pb[i] = add_tensor(T, nm, 1, 3);
    }
    T->o_sstab = T->stab ? add_tensor(T, "syn.stab", 3, T->L) : -1;
    /* buffers */
    const size_t nl = (size_t)T->n_lat, np = (size_t)T->n_par, npix = (size_t)T->npix;
    T->y = zalloc(nl); T->yg = zalloc(nl); T->lm = zalloc(nl); T->lv = zalloc(nl);
    T->th1 = zalloc(nl); T->th2 = zalloc(nl);
    T->q = (int32_t*)calloc(nl, sizeof(int32_t));
    T->par = zalloc(np); T->grad = zalloc(np); T->nm = zalloc(np); T->nv = zalloc(np);
    for (int i = 0; i < n; ++i) {
        T->stride[i] = T->g[i].cols + 2 * T->P;
        const size_t sz = (size_t)(T->g[i].rows + 2 * T->P) * T->stride[i];
        T->pv[i] = zalloc(sz);
        T->pg[i] = zalloc(sz);
    }
    T->z = zalloc((size_t)T->L * npix);
    T->dz = zalloc((size_t)T->L * npix);
    T->h1 = zalloc((size_t)T->synF * npix);
    T->trunk = zalloc(3 * npix);
    T->post[0] = zalloc(3 * npix);
    T->post[1] = zalloc(3 * npix);
    T->xhat = zalloc(3 * npix);
    T->dx = zalloc(3 * npix);
    for (int k = 1; k < T->L; ++k)
        for (int j = k - 1; j >= 0; --j) {
            const int ri = cdiv(T->H, 1 << (j + 1)), ro = cdiv(T->H, 1 << j), co = cdiv(T->W, 1 << j);
            T->ups_row[k][j] = zalloc((size_t)ri * co);
            T->ups_col[k][j] = zalloc((size_t)ro * co);
            T->ups_out[k][j] = j == 0 ? T->z + (size_t)k * npix : zalloc((size_t)ro * co);
        }
    return CC_OK;
}

static float* PV(cc_trainer* T, int gi, int r, int c) {
    return T->pv[gi] + (size_t)(r + T->P) * T->stride[gi] + (c + T->P);
}
static float* PG(cc_trainer* T, int gi, int r, int c) {
    return T->pg[gi] + (size_t)(r + T->P) * T->stride[gi] + (c + T->P);
}

/* ------------------------------------------------ rate_pass (per latent) --
 * entropy_model.hpp:180-336.  upstream = lambda/npix; bwd when upstream != 0;
 * latent_grads selects the pads-gradient outputs (off in hardround). */
static double rate_pass(cc_trainer* T, float upstream, int latent_grads) {
    const int D = T->D, Wd = T->Wd, S = T->S;
    const float* w1 = T->par + T->o_l1w;
    const float* b1 = T->par + T->o_l1b;
    const float* w2 = T->par + T->o_l2w;
    const float* b2 = T->par + T->o_l2b;
    const float* w3 = T->par + T->o_hw;
    const float* b3 = T->par + T->o_hb;
    const float* st = T->stab ? T->par + T->o_astab : NULL;
    float* dw1 = T->grad + T->o_l1w;
    float* db1 = T->grad + T->o_l1b;
    float* dw2 = T->grad + T->o_l2w;
    float* db2 = T->grad + T->o_l2b;
    float* dw3 = T->grad + T->o_hw;
    float* db3 = T->grad + T->o_hb;
    float* dst = T->stab ? T->grad + T->o_astab : NULL;
    const int bwd = upstream != 0.0f;
    float C[200], H1[64], H2[64], R[16], dH2[64], dH1[64], dC[200];
    double total = 0.0;
    for (int gi = 0; gi < T->n_grids; ++gi) {
        const Grid* g = &T->g[gi];
        const int slot = g->slot, rd = g->rdim;
        const float* wf = slot >= 0 ? T->par + T->o_ifw[slot] : NULL;
        const float* bf = slot >= 0 ? T->par + T->o_ifb[slot] : NULL;
        float* dwf = slot >= 0 ? T->grad + T->o_ifw[slot] : NULL;
        float* dbf = slot >= 0 ? T->grad + T->o_ifb[slot] : NULL;
        for (int r = 0; r < g->rows; ++r)
            for (int c = 0; c < g->cols; ++c) {
                /* context gather :233-248 (borders of the padded grid are 0) */
                for (int o = 0; o < S; ++o) C[o] = *PV(T, gi, r + T->ctx_dy[o], c + T->ctx_dx[o]);
                for (int f = 0; f < T->F; ++f) C[S + f] = 0.0f;
                if (slot >= 0) {
                    for (int j = 0; j < rd; ++j) {
                        const int sh = T->g[j].level - g->level;
                        R[j] = *PV(T, j, r >> sh, c >> sh);
                    }
                    for (int f = 0; f < T->F; ++f) {
                        float a = bf[f];
                        for (int j = 0; j < rd; ++j) a += R[j] * wf[f * rd + j];
                        C[S + f] = a;
                    }
                }
                /* MLP :250-255 */
                for (int a = 0; a < Wd; ++a) {
                    float acc = b1[a];
                    for (int k = 0; k < D; ++k) acc += C[k] * w1[a * D + k];
                    H1[a] = acc > 0.0f ? acc : 0.0f;
                }
                for (int a = 0; a < Wd; ++a) {
                    float acc = b2[a];
                    for (int k = 0; k < Wd; ++k) acc += H1[k] * w2[a * Wd + k];
                    H2[a] = acc > 0.0f ? acc : 0.0f;
                }
                float raw[2];
                for (int j = 0; j < 2; ++j) {
                    float acc = b3[j];
                    for (int k = 0; k < Wd; ++k) acc += H2[k] * w3[j * Wd + k];
                    if (st)
                        for (int k = 0; k < D; ++k) acc += C[k] * st[j * D + k];
                    raw[j] = acc;
                }
                /* Laplace :257-273 */
                const float v = *PV(T, gi, r, c);
                const float mu = raw[0];
                const float sg = fminr(SIGMA_MAX, fmaxr(SIGMA_MIN, cc_exp(raw[1])));
                const float b = sg * INV_SQRT2;
                const float u = fabsf(v - mu);
                const float e1 = cc_exp(-(u + 0.5f) / b);
                const float e2 = cc_exp(-fabsf(u - 0.5f) / b);
                const float p = u >= 0.5f ? 0.5f * (e2 - e1) : 1.0f - 0.5f * (e1 + e2);
                total += (double)(-(cc_log(fmaxr(p, PFLOOR)) * 1.4426950408889634f));
                if (!bwd) continue;
                /* rate backward :276-296 */
                float dmu = 0.0f, dsr = 0.0f;
                if (p > PFLOOR) {
                    const float t = v - mu;
                    const float dbits_dp = -1.0f / (p * 0.6931471805599453f);
                    const float dp_du = (e1 - e2) / (2.0f * b);
                    const float sgn = t > 0.0f ? 1.0f : (t < 0.0f ? -1.0f : 0.0f);
                    const float dp_db = -((u + 0.5f) * e1 - (u - 0.5f) * e2) / (2.0f * b * b);
                    const float up = upstream * dbits_dp;
                    dmu = -up * dp_du * sgn;
                    if (sg > SIGMA_MIN && sg < SIGMA_MAX) dsr = up * dp_db * INV_SQRT2 * sg;
                    if (latent_grads) *PG(T, gi, r, c) += up * dp_du * sgn;
                }
                /* MLP backward :298-310 */
                for (int a = 0; a < Wd; ++a) {
                    const float d = dmu * w3[a] + dsr * w3[Wd + a];
                    dH2[a] = H2[a] > 0.0f ? d : 0.0f;
                }
                for (int k = 0; k < Wd; ++k) {
                    dw3[k] += dmu * H2[k];
                    dw3[Wd + k] += dsr * H2[k];
                }
                db3[0] += dmu;
                db3[1] += dsr;
                for (int k = 0; k < Wd; ++k) {
                    float acc = 0.0f;
                    for (int a = 0; a < Wd; ++a) acc += dH2[a] * w2[a * Wd + k];
                    dH1[k] = H1[k] > 0.0f ? acc : 0.0f;
                }
                for (int a = 0; a < Wd; ++a) {
                    for (int k = 0; k < Wd; ++k) dw2[a * Wd + k] += dH2[a] * H1[k];
                    db2[a] += dH2[a];
                }
                for (int k = 0; k < D; ++k) {
                    float acc = 0.0f;
                    for (int a = 0; a < Wd; ++a) acc += dH1[a] * w1[a * D + k];
                    if (st) acc += dmu * st[k] + dsr * st[D + k];
                    dC[k] = acc;
                }
                for (int a = 0; a < Wd; ++a) {
                    for (int k = 0; k < D; ++k) dw1[a * D + k] += dH1[a] * C[k];
                    db1[a] += dH1[a];
                }
                if (st)
                    for (int k = 0; k < D; ++k) {
                        dst[k] += dmu * C[k];
                        dst[D + k] += dsr * C[k];
                    }
                /* context-gradient scatter :312-317 */
                if (latent_grads)
                    for (int o = 0; o < S; ++o) *PG(T, gi, r + T->ctx_dy[o], c + T->ctx_dx[o]) += dC[o];
                /* IFCE backward :318-332 */
                if (slot >= 0) {
                    for (int f = 0; f < T->F; ++f) {
                        const float dF = dC[S + f];
                        for (int j = 0; j < rd; ++j) dwf[f * rd + j] += dF * R[j];
                        dbf[f] += dF;
                    }
                    if (latent_grads)
                        for (int j = 0; j < rd; ++j) {
                            float acc = 0.0f;
                            for (int f = 0; f < T->F; ++f) acc += dC[S + f] * wf[f * rd + j];
                            const int sh = T->g[j].level - g->level;
                            *PG(T, j, r >> sh, c >> sh) += acc;
                        }
                }
            }
    }
    return total;
}

/* ------------------------------------------ upsampling (synthesis.hpp) --- */
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
/* tap table of the symmetric x2 transposed conv (layers.hpp:346-351) */
static void tmap(int t, int last, int* idx, int* tap) {
    const int u = t >> 1;
    if ((t & 1) == 0) {
        idx[0] = u >= 2 ? u - 2 : 0; idx[1] = u >= 1 ? u - 1 : 0; idx[2] = u; idx[3] = u < last ? u + 1 : last;
        tap[0] = 0; tap[1] = 2; tap[2] = 3; tap[3] = 1;
    } else {
        idx[0] = u >= 1 ? u - 1 : 0; idx[1] = u; idx[2] = u < last ? u + 1 : last; idx[3] = u + 2 < last ? u + 2 : last;
        tap[0] = 1; tap[1] = 3; tap[2] = 2; tap[3] = 0;
    }
}

/* stage input of grid k at stage j: the padded main grid or the previous stage */
static const float* stage_in(cc_trainer* T, int k, int j, int* stride) {
    if (j == k - 1) {
        *stride = T->stride[T->main_gi[k]];
        return PV(T, T->main_gi[k], 0, 0);
    }
    *stride = cdiv(T->W, 1 << (j + 1));
    return T->ups_out[k][j + 1];
}

static void upsample_forward(cc_trainer* T) { /* synthesis.hpp:55-93 */
    const Grid* g0 = &T->g[T->main_gi[0]];
    for (int r = 0; r < g0->rows; ++r)
        for (int c = 0; c < g0->cols; ++c) T->z[(size_t)r * T->W + c] = *PV(T, T->main_gi[0], r, c);
    for (int k = 1; k < T->L; ++k)
        for (int j = k - 1; j >= 0; --j) {
            const float* k4 = T->par + T->o_tc[j];
            const float* r3 = T->par + T->o_rf[j];
            int ins;
            const float* in = stage_in(T, k, j, &ins);
            const int ri = cdiv(T->H, 1 << (j + 1)), ci = cdiv(T->W, 1 << (j + 1));
            const int ro = cdiv(T->H, 1 << j), co = cdiv(T->W, 1 << j);
            float* row = T->ups_row[k][j];
            float* col = T->ups_col[k][j];
            float* out = T->ups_out[k][j];
            int idx[4], tap[4];
            for (int r = 0; r < ri; ++r) /* tconv2x_rows_forward layers.hpp:353-376 */
                for (int t = 0; t < co; ++t) {
                    tmap(t, ci - 1, idx, tap);
                    const float* x = in + (size_t)r * ins;
                    row[(size_t)r * co + t] = k4[tap[0]] * x[idx[0]] + k4[tap[1]] * x[idx[1]] +
                                              k4[tap[2]] * x[idx[2]] + k4[tap[3]] * x[idx[3]];
                }
            for (int t = 0; t < ro; ++t) { /* tconv2x_cols_forward :407-429 */
                tmap(t, ri - 1, idx, tap);
                for (int c = 0; c < co; ++c)
                    col[(size_t)t * co + c] = k4[tap[0]] * row[(size_t)idx[0] * co + c] +
                                              k4[tap[1]] * row[(size_t)idx[1] * co + c] +
                                              k4[tap[2]] * row[(size_t)idx[2] * co + c] +
                                              k4[tap[3]] * row[(size_t)idx[3] * co + c];
            }
            for (int r = 0; r < ro; ++r) /* conv3x3_sym_forward :467-483 */
                for (int c = 0; c < co; ++c) {
                    const int rm = clampi(r - 1, 0, ro - 1), rp = clampi(r + 1, 0, ro - 1);
                    const int cm = clampi(c - 1, 0, co - 1), cp = clampi(c + 1, 0, co - 1);
                    const float* x0 = col + (size_t)rm * co;
                    const float* x1 = col + (size_t)r * co;
                    const float* x2 = col + (size_t)rp * co;
                    out[(size_t)r * co + c] = r3[0] * x1[c] + r3[1] * (x0[c] + x2[c] + x1[cm] + x1[cp]) +
                                              r3[2] * (x0[cm] + x0[cp] + x2[cm] + x2[cp]);
                }
        }
}

static void upsample_backward(cc_trainer* T) { /* synthesis.hpp:103-139 */
    const int npix = (int)T->npix;
    const Grid* g0 = &T->g[T->main_gi[0]];
    for (int r = 0; r < g0->rows; ++r)
        for (int c = 0; c < g0->cols; ++c) *PG(T, T->main_gi[0], r, c) += T->dz[(size_t)r * T->W + c];
    for (int k = 1; k < T->L; ++k) {
        float* dcur = NULL;
        for (int j = 0; j <= k - 1; ++j) {
            const float* k4 = T->par + T->o_tc[j];
            const float* r3 = T->par + T->o_rf[j];
            float* dk4 = T->grad + T->o_tc[j];
            float* dr3 = T->grad + T->o_rf[j];
            const int ri = cdiv(T->H, 1 << (j + 1)), ci = cdiv(T->W, 1 << (j + 1));
            const int ro = cdiv(T->H, 1 << j), co = cdiv(T->W, 1 << j);
            const float* dout = j == 0 ? T->dz + (size_t)k * npix : dcur;
            const float* col = T->ups_col[k][j];
            const float* row = T->ups_row[k][j];
            /* conv3x3_sym_backward :486-515 */
            float* dcol = zalloc((size_t)ro * co);
            double ac = 0.0, ae = 0.0, ao = 0.0;
            for (int r = 0; r < ro; ++r)
                for (int c = 0; c < co; ++c) {
                    const int rm = clampi(r - 1, 0, ro - 1), rp = clampi(r + 1, 0, ro - 1);
                    const int cm = clampi(c - 1, 0, co - 1), cp = clampi(c + 1, 0, co - 1);
                    const float* x0 = col + (size_t)rm * co;
                    const float* x1 = col + (size_t)r * co;
                    const float* x2 = col + (size_t)rp * co;
                    const float g = dout[(size_t)r * co + c];
                    ac += (double)g * (double)x1[c];
                    ae += (double)g * (double)(x0[c] + x2[c] + x1[cm] + x1[cp]);
                    ao += (double)g * (double)(x0[cm] + x0[cp] + x2[cm] + x2[cp]);
                    float* d0 = dcol + (size_t)rm * co;
                    float* d1 = dcol + (size_t)r * co;
                    float* d2 = dcol + (size_t)rp * co;
                    d1[c] += r3[0] * g;
                    d0[c] += r3[1] * g; d2[c] += r3[1] * g; d1[cm] += r3[1] * g; d1[cp] += r3[1] * g;
                    d0[cm] += r3[2] * g; d0[cp] += r3[2] * g; d2[cm] += r3[2] * g; d2[cp] += r3[2] * g;
                }
            dr3[0] += (float)ac;
            dr3[1] += (float)ae;
            dr3[2] += (float)ao;
            /* tconv2x_cols_backward :432-460 */
            float* drow = zalloc((size_t)ri * co);
            int idx[4], tap[4];
            for (int t = 0; t < ro; ++t) {
                tmap(t, ri - 1, idx, tap);
                for (int q = 0; q < 4; ++q) {
                    double acc = 0.0;
                    for (int c = 0; c < co; ++c) {
                        const float g = dcol[(size_t)t * co + c];
                        drow[(size_t)idx[q] * co + c] += k4[tap[q]] * g;
                        acc += (double)g * (double)row[(size_t)idx[q] * co + c];
                    }
                    dk4[tap[q]] += (float)acc;
                }
            }
            /* tconv2x_rows_backward :378-405 */
            int ins;
            const float* in = stage_in(T, k, j, &ins);
            float* dprev = zalloc((size_t)ri * ci);
            for (int r = 0; r < ri; ++r)
                for (int t = 0; t < co; ++t) {
                    tmap(t, ci - 1, idx, tap);
                    const float g = drow[(size_t)r * co + t];
                    for (int q = 0; q < 4; ++q) {
                        dprev[(size_t)r * ci + idx[q]] += k4[tap[q]] * g;
                        dk4[tap[q]] += g * in[(size_t)r * ins + idx[q]];
                    }
                }
            free(dcol);
            free(drow);
            if (dcur) free(dcur);
            dcur = dprev;
        }
        const int gi = T->main_gi[k];
        for (int r = 0; r < T->g[gi].rows; ++r)
            for (int c = 0; c < T->g[gi].cols; ++c) *PG(T, gi, r, c) += dcur[(size_t)r * T->g[gi].cols + c];
        free(dcur);
    }
}

/* ------------------------------------------ synthesis (synthesis.hpp) ---- */
static void synth_forward(cc_trainer* T) { /* :191-213 */
    const size_t np = (size_t)T->npix;
    const int L = T->L, F = T->synF;
    const float* c1w = T->par + T->o_c1w;
    const float* c1b = T->par + T->o_c1b;
    const float* c2w = T->par + T->o_c2w;
    const float* c2b = T->par + T->o_c2b;
    for (size_t p = 0; p < np; ++p) {
        for (int f = 0; f < F; ++f) {
            float acc = c1b[f];
            for (int k = 0; k < L; ++k) acc += c1w[f * L + k] * T->z[k * np + p];
            T->h1[f * np + p] = acc > 0.0f ? acc : 0.0f;
        }
        for (int co = 0; co < 3; ++co) {
            float acc = c2b[co];
            for (int f = 0; f < F; ++f) acc += c2w[co * F + f] * T->h1[f * np + p];
            T->trunk[co * np + p] = acc;
        }
    }
    const float* cur = T->trunk;
    for (int i = 0; i < T->posts; ++i) { /* conv3x3_forward layers.hpp:257-300 + residual */
        const float* w = T->par + T->o_pw[i];
        const float* b = T->par + T->o_pb[i];
        for (int co = 0; co < 3; ++co)
            for (int r = 0; r < T->H; ++r)
                for (int c = 0; c < T->W; ++c) {
                    float acc = b[co];
                    for (int ci = 0; ci < 3; ++ci) {
                        const float* k = w + (co * 3 + ci) * 9;
                        float s = 0.0f;
                        for (int dr = -1; dr <= 1; ++dr)
                            for (int dc = -1; dc <= 1; ++dc) {
                                const int rr = clampi(r + dr, 0, T->H - 1), cc = clampi(c + dc, 0, T->W - 1);
                                s += k[(dr + 1) * 3 + (dc + 1)] * cur[ci * np + (size_t)rr * T->W + cc];
                            }
                        acc += s;
                    }
                    T->post[i][co * np + (size_t)r * T->W + c] = acc + cur[co * np + (size_t)r * T->W + c];
                }
        cur = T->post[i];
    }
    for (size_t e = 0; e < 3 * np; ++e) T->xhat[e] = cur[e];
    if (T->stab) {
        const float* s = T->par + T->o_sstab;
        for (int co = 0; co < 3; ++co)
            for (int k = 0; k < L; ++k)
                for (size_t p = 0; p < np; ++p) T->xhat[co * np + p] += s[co * L + k] * T->z[k * np + p];
    }
    for (size_t e = 0; e < 3 * np; ++e) T->xhat[e] = fminr(1.0f, fmaxr(0.0f, T->xhat[e]));
}

static void synth_backward(cc_trainer* T) { /* :216-233 */
    const size_t np = (size_t)T->npix;
    const int L = T->L, F = T->synF;
    memset(T->dz, 0, sizeof(float) * (size_t)L * np);
    if (T->stab) {
        const float* s = T->par + T->o_sstab;
        float* ds = T->grad + T->o_sstab;
        for (int co = 0; co < 3; ++co)
            for (int k = 0; k < L; ++k) {
                double acc = 0.0;
                for (size_t p = 0; p < np; ++p) {
                    T->dz[k * np + p] += s[co * L + k] * T->dx[co * np + p];
                    acc += (double)T->dx[co * np + p] * (double)T->z[k * np + p];
                }
                ds[co * L + k] += (float)acc;
            }
    }
    float* dcur = zalloc(3 * np);
    memcpy(dcur, T->dx, sizeof(float) * 3 * np);
    for (int i = T->posts - 1; i >= 0; --i) { /* conv3x3_backward :302-343 */
        const float* in = i > 0 ? T->post[i - 1] : T->trunk;
        const float* w = T->par + T->o_pw[i];
        float* dw = T->grad + T->o_pw[i];
        float* db = T->grad + T->o_pb[i];
        float* dprev = zalloc(3 * np);
        for (int co = 0; co < 3; ++co) {
            double bacc = 0.0;
            for (int r = 0; r < T->H; ++r)
                for (int c = 0; c < T->W; ++c) {
                    const float g = dcur[co * np + (size_t)r * T->W + c];
                    bacc += (double)g;
                    for (int ci = 0; ci < 3; ++ci)
                        for (int dr = -1; dr <= 1; ++dr)
                            for (int dc = -1; dc <= 1; ++dc) {
                                const int rr = clampi(r + dr, 0, T->H - 1), cc = clampi(c + dc, 0, T->W - 1);
                                const int tap = (co * 3 + ci) * 9 + (dr + 1) * 3 + (dc + 1);
                                dprev[ci * np + (size_t)rr * T->W + cc] += w[tap] * g;
                                dw[tap] += g * in[ci * np + (size_t)rr * T->W + cc];
                            }
                }
            db[co] += (float)bacc;
        }
        for (size_t e = 0; e < 3 * np; ++e) dprev[e] += dcur[e];
        free(dcur);
        dcur = dprev;
    }
    const float* c1w = T->par + T->o_c1w;
    const float* c2w = T->par + T->o_c2w;
    float* dc1w = T->grad + T->o_c1w;
    float* dc1b = T->grad + T->o_c1b;
    float* dc2w = T->grad + T->o_c2w;
    float* dc2b = T->grad + T->o_c2b;
    /* c2 backward (conv1x1_backward :216-250), relu mask, c1 backward */
    for (int co = 0; co < 3; ++co) {
        double b = 0.0;
        for (size_t p = 0; p < np; ++p) b += (double)dcur[co * np + p];
        dc2b[co] += (float)b;
        for (int f = 0; f < F; ++f) {
            double a = 0.0;
            for (size_t p = 0; p < np; ++p) a += (double)dcur[co * np + p] * (double)T->h1[f * np + p];
            dc2w[co * F + f] += (float)a;
        }
    }
    float* dh1 = zalloc((size_t)F * np);
    for (int f = 0; f < F; ++f)
        for (size_t p = 0; p < np; ++p) {
            float a = 0.0f;
            for (int co = 0; co < 3; ++co) a += c2w[co * F + f] * dcur[co * np + p];
            dh1[f * np + p] = T->h1[f * np + p] > 0.0f ? a : 0.0f;
        }
    for (int f = 0; f < F; ++f) {
        double b = 0.0;
        for (size_t p = 0; p < np; ++p) b += (double)dh1[f * np + p];
        dc1b[f] += (float)b;
        for (int k = 0; k < L; ++k) {
            double a = 0.0;
            for (size_t p = 0; p < np; ++p) a += (double)dh1[f * np + p] * (double)T->z[k * np + p];
            dc1w[f * L + k] += (float)a;
        }
    }
    for (int k = 0; k < L; ++k)
        for (size_t p = 0; p < np; ++p) {
            float a = 0.0f;
            for (int f = 0; f < F; ++f) a += c1w[f * L + k] * dh1[f * np + p];
            T->dz[k * np + p] += a;
        }
    free(dh1);
    free(dcur);
}

/* synth_forward_backward (encoder.hpp:245-272) */
static double synth_fb(cc_trainer* T, int forward_only) {
    upsample_forward(T);
    synth_forward(T);
    const size_t n = 3 * (size_t)T->npix;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = (double)T->xhat[i] - (double)T->img[i];
        acc += d * d;
    }
    const double mse = acc / (double)n;
    if (forward_only || !isfinite(mse)) return mse;
    const float s = (float)(2.0 / (double)n);
    for (size_t i = 0; i < n; ++i) T->dx[i] = s * (T->xhat[i] - T->img[i]);
    synth_backward(T);
    upsample_backward(T);
    return mse;
}

/* ------------------------------------------------------- optimizers ------ */
static int adam_step(float* p, const float* g, size_t n, float* m, float* v, int64_t* t, double lr) {
    for (size_t i = 0; i < n; ++i) /* optim.hpp:38-53 */
        if (!isfinite(g[i])) return 0;
    *t += 1;
    const double bc1 = 1.0 - pow(0.9, (double)*t), bc2 = 1.0 - pow(0.999, (double)*t);
    for (size_t i = 0; i < n; ++i) {
        const double gi = (double)g[i];
        const double mt = 0.9 * (double)m[i] + (1.0 - 0.9) * gi;
        const double vt = 0.999 * (double)v[i] + (1.0 - 0.999) * gi * gi;
        m[i] = (float)mt;
        v[i] = (float)vt;
        p[i] = (float)((double)p[i] - lr * (mt / bc1) / (sqrt(vt / bc2) + 1e-8));
    }
    return 1;
}

static void zero_all_grads(cc_trainer* T) { /* encoder.hpp:237-241 */
    memset(T->grad, 0, sizeof(float) * (size_t)T->n_par);
    memset(T->yg, 0, sizeof(float) * (size_t)T->n_lat);
    for (int gi = 0; gi < T->n_grids; ++gi)
        memset(T->pg[gi], 0, sizeof(float) * (size_t)(T->g[gi].rows + 2 * T->P) * T->stride[gi]);
}

static double rd(double mse, double bits, double npix, double lam) { return mse + lam * (bits / npix); }

static double proxy_iteration(cc_trainer* T, double lr, double temp, double noise) { /* encoder.hpp:97-135 */
    const float tf = (float)temp, nf = (float)noise;
    zero_all_grads(T);
    const float inv_denom = 1.0f / softround_denom(tf), inv_t = 1.0f / tf;
    for (int gi = 0; gi < T->n_grids; ++gi) { /* soft_quantize_forward latent.hpp:120-128 */
        const Grid* g = &T->g[gi];
        const uint64_t stream = hash_combine(hash_combine(T->enc.seed, (uint64_t)T->global_iter), (uint64_t)gi);
        for (int r = 0; r < g->rows; ++r)
            for (int c = 0; c < g->cols; ++c) {
                const size_t li = (size_t)r * g->cols + c;
                const float x = T->y[g->off + li];
                float f = floorf(x);
                const float t1 = cc_tanh((x - f - 0.5f) * inv_t);
                float o = f + 0.5f + t1 * inv_denom;
                if (nf > 0.0f) o += nf * counter_gauss(stream, li);
                f = floorf(o);
                const float t2 = cc_tanh((o - f - 0.5f) * inv_t);
                *PV(T, gi, r, c) = f + 0.5f + t2 * inv_denom;
                T->th1[g->off + li] = t1;
                T->th2[g->off + li] = t2;
            }
    }
    const float upstream = (float)(T->enc.lambda / (double)T->npix);
    const double bits = rate_pass(T, upstream, 1);
    const double mse = synth_fb(T, 0);
    const double cost = rd(mse, bits, (double)T->npix, T->enc.lambda);
    T->last_mse = mse;
    T->last_bits = bits;
    if (!isfinite(cost)) return cost;
    const float scale = 1.0f / (tf * softround_denom(tf));
    for (int gi = 0; gi < T->n_grids; ++gi) { /* soft_quantize_backward latent.hpp:131-139 */
        const Grid* g = &T->g[gi];
        for (int r = 0; r < g->rows; ++r)
            for (int c = 0; c < g->cols; ++c) {
                const size_t i = g->off + (size_t)r * g->cols + c;
                const float d2 = fmaf(-T->th2[i], T->th2[i], 1.0f) * scale;
                const float d1 = fmaf(-T->th1[i], T->th1[i], 1.0f) * scale;
                T->yg[i] += *PG(T, gi, r, c) * d2 * d1;
            }
        if (!adam_step(T->y + g->off, T->yg + g->off, (size_t)g->rows * g->cols, T->lm + g->off,
                       T->lv + g->off, &T->lat_t[gi], lr))
            ++T->skipped;
    }
    for (int ti = 0; ti < T->n_t; ++ti) /* NnOptimizer::step optim.hpp:277-286 (Adam) */
        if (!adam_step(T->par + T->t[ti].off, T->grad + T->t[ti].off, (size_t)T->t[ti].size,
                       T->nm + T->t[ti].off, T->nv + T->t[ti].off, &T->nn_t[ti], lr))
            ++T->skipped;
    ++T->global_iter;
    return cost;
}

static void snapshot_take(cc_trainer* T, int slot, double cost) {
    Snap* s = &T->snaps[slot];
    if (!s->y) {
        s->y = zalloc((size_t)T->n_lat);
        s->p = zalloc((size_t)T->n_par);
    }
    memcpy(s->y, T->y, sizeof(float) * (size_t)T->n_lat);
    memcpy(s->p, T->par, sizeof(float) * (size_t)T->n_par);
    s->cost = cost;
    s->valid = 1;
}

static double hardround_iteration(cc_trainer* T, double lr, int best) { /* encoder.hpp:141-155 */
    zero_all_grads(T);
    const float upstream = (float)(T->enc.lambda / (double)T->npix);
    const double bits = rate_pass(T, upstream, 0);
    const double mse = synth_fb(T, 0);
    const double cost = rd(mse, bits, (double)T->npix, T->enc.lambda);
    T->last_mse = mse;
    T->last_bits = bits;
    if (!isfinite(cost)) return cost;
    if (best >= 0) {
        const double bc = T->snaps[best].valid ? T->snaps[best].cost : INFINITY;
        if (cost < bc) snapshot_take(T, best, cost);
    }
    for (int ti = 0; ti < T->n_t; ++ti)
        if (!adam_step(T->par + T->t[ti].off, T->grad + T->t[ti].off, (size_t)T->t[ti].size,
                       T->nm + T->t[ti].off, T->nv + T->t[ti].off, &T->nn_t[ti], lr))
            ++T->skipped;
    ++T->global_iter;
    return cost;
}

static void quantize_all(cc_trainer* T) {
    for (int64_t i = 0; i < T->n_lat; ++i) T->q[i] = quantize_value(T->y[i], 255);
}
static void load_pads_from_q(cc_trainer* T) { /* encoder.hpp:170-180 */
    for (int gi = 0; gi < T->n_grids; ++gi)
        for (int r = 0; r < T->g[gi].rows; ++r)
            for (int c = 0; c < T->g[gi].cols; ++c)
                *PV(T, gi, r, c) = (float)T->q[T->g[gi].off + (size_t)r * T->g[gi].cols + c];
}
static double true_cost(cc_trainer* T, double* psnr, double* bpp) { /* encoder.hpp:158-168 */
    quantize_all(T);
    load_pads_from_q(T);
    const double bits = rate_pass(T, 0.0f, 0);
    const double mse = synth_fb(T, 1);
    if (psnr) *psnr = mse > 0 ? fmin(99.0, -10.0 * log10(mse)) : 99.0;
    if (bpp) *bpp = bits / (double)T->npix;
    return rd(mse, bits, (double)T->npix, T->enc.lambda);
}

static void reset_optimizers(cc_trainer* T) {
    memset(T->lm, 0, sizeof(float) * (size_t)T->n_lat);
    memset(T->lv, 0, sizeof(float) * (size_t)T->n_lat);
    memset(T->nm, 0, sizeof(float) * (size_t)T->n_par);
    memset(T->nv, 0, sizeof(float) * (size_t)T->n_par);
    memset(T->lat_t, 0, sizeof(T->lat_t));
    memset(T->nn_t, 0, sizeof(T->nn_t));
}

static void zero_pads(cc_trainer* T) {
    for (int gi = 0; gi < T->n_grids; ++gi)
        memset(T->pv[gi], 0, sizeof(float) * (size_t)(T->g[gi].rows + 2 * T->P) * T->stride[gi]);
}

static void fresh_candidate(cc_trainer* T, int index) { /* encoder.hpp:82-93 */
    const uint64_t ls = hash_combine(T->enc.seed, (uint64_t)(0x1000 + index));
    for (int gi = 0; gi < T->n_grids; ++gi) { /* init_latents_uniform latent.hpp:73-80 */
        const uint64_t gs = hash_combine(ls, (uint64_t)gi);
        for (int64_t i = 0; i < (int64_t)T->g[gi].rows * T->g[gi].cols; ++i)
            T->y[T->g[gi].off + i] = counter_uniform(gs, (uint64_t)i, -0.3f, 0.3f);
    }
    memset(T->par, 0, sizeof(float) * (size_t)T->n_par);
    const uint64_t ms = hash_combine(T->enc.seed, (uint64_t)(0x2000 + index));
    uint64_t ctr = 0;
#define KAIMING(off, n, fan) do { const uint64_t s_ = hash_combine(ms, ctr++); \
        const float a_ = sqrtf(6.0f / (float)(fan)); \
        for (int i_ = 0; i_ < (n); ++i_) T->par[(off) + i_] = counter_uniform(s_, (uint64_t)i_, -a_, a_); } while (0)
    KAIMING(T->o_l1w, T->Wd * T->D, T->D); /* init_model model.hpp:137-156 */
    KAIMING(T->o_l2w, T->Wd * T->Wd, T->Wd);
    KAIMING(T->o_hw, 2 * T->Wd, T->Wd);
    for (int s = 0; s < T->n_slots; ++s) {
        const int rd = T->g[T->slot_gi[s]].rdim;
        KAIMING(T->o_ifw[s], T->F * rd, rd);
    }
    static const float bic[4] = {-0.0234375f, -0.0703125f, 0.2265625f, 0.8671875f};
    for (int j = 0; j < T->L - 1; ++j) {
        for (int i = 0; i < 4; ++i) T->par[T->o_tc[j] + i] = bic[i];
        T->par[T->o_rf[j]] = 1.0f;
    }
    KAIMING(T->o_c1w, T->synF * T->L, T->L);
    KAIMING(T->o_c2w, 3 * T->synF, T->synF);
#undef KAIMING
    reset_optimizers(T);
    zero_pads(T);
    T->loaded = 1;
    T->cur_cost = INFINITY;
}

/* ----------------------------------------------------------- the ABI ---- */
const char* cc_last_error(void) { return g_err; }
const char* cc_impl_name(void) { return "port"; }

int cc_decoder_config_preset(const char* name, cc_decoder_config* out) {
    static const cc_decoder_config pres[4] = {{0, 6, 2, 8, 2, 8, 1, 1, 1}, {1, 10, 4, 10, 2, 16, 2, 1, 1},
                                              {2, 14, 6, 20, 2, 48, 2, 1, 1}, {3, 20, 6, 26, 2, 64, 2, 1, 1}};
    static const char* names[4] = {"lop", "mop", "hop", "vhop"};
    for (int i = 0; i < 4; ++i)
        if (name && strcmp(name, names[i]) == 0) {
            *out = pres[i];
            return CC_OK;
        }
    return fail(CC_ERR_CONFIG, "unknown decoder config");
}

int cc_encoder_config_default(cc_encoder_config* o) {
    memset(o, 0, sizeof(*o));
    o->warmup_candidates = 5; o->warmup_keep = 2; o->warmup_iters = 400; o->main_iters = 96700;
    o->hardround_iters = 500; o->lr_start = 1e-2; o->lr_end = 1e-6; o->noise_std_start = 0.22;
    o->noise_std_end = 0.15; o->temp_start = 0.35; o->temp_end = 0.08; o->hardround_lr = 1e-4;
    o->lambda = 0.001; o->seed = 0; o->use_soap = 0; o->true_cost_interval = 1000;
    return CC_OK;
}

int cc_encoder_config_with_total(int total, cc_encoder_config* o) { /* config.hpp:127-141 */
    cc_encoder_config_default(o);
    if (total == 100000) return CC_OK;
    if (total < 20) return fail(CC_ERR_CONFIG, "iteration budget too small");
    const double f = (double)total / 100000.0;
    o->warmup_iters = (int)lround(400.0 * f) > 1 ? (int)lround(400.0 * f) : 1;
    o->hardround_iters = (int)lround(500.0 * f) > 1 ? (int)lround(500.0 * f) : 1;
    int rest = total - (o->warmup_candidates + o->warmup_keep) * o->warmup_iters - o->hardround_iters;
    while (rest < 1 && o->warmup_iters > 1) {
        --o->warmup_iters;
        rest = total - (o->warmup_candidates + o->warmup_keep) * o->warmup_iters - o->hardround_iters;
    }
    o->main_iters = rest > 1 ? rest : 1;
    return CC_OK;
}

double cc_count_macs_per_pixel(const cc_decoder_config* cfg, int H, int W) { /* synthesis.hpp:239-277 */
    const int L = (int64_t)H * W < 1000000 ? 7 : 8;
    const double npix = (double)H * W;
    const int d = cfg->spatial_ctx + cfg->ifce_dim, w = cfg->arm_width;
    double arm = (double)d * w + (double)w * w + 2.0 * w + (cfg->use_stabilizer ? 2.0 * d : 0.0);
    double tot = 0.0;
    for (int k = 0; k < L; ++k) tot += (double)cdiv(H, 1 << k) * cdiv(W, 1 << k) * arm;
    if (cfg->use_hyperlatents)
        for (int k = 4; k < L; ++k) tot += (double)cdiv(H, 1 << k) * cdiv(W, 1 << k) * arm;
    if (cfg->ifce_dim > 0)
        for (int k = 0; k < 3 && k < L; ++k)
            tot += (double)cdiv(H, 1 << k) * cdiv(W, 1 << k) *
                   (double)((cfg->use_hyperlatents ? L - 4 : 0) + L - 1 - k) * cfg->ifce_dim;
    for (int k = 1; k < L; ++k)
        for (int j = k - 1; j >= 0; --j)
            tot += (double)cdiv(H, 1 << (j + 1)) * cdiv(W, 1 << j) * 4.0 +
                   (double)cdiv(H, 1 << j) * cdiv(W, 1 << j) * 13.0;
    double syn = (double)L * cfg->synth_hidden + cfg->synth_hidden * 3.0 + cfg->synth_posts * 81.0;
    if (cfg->use_stabilizer) syn += 3.0 * L;
    return (tot + npix * syn) / npix;
}

int cc_make_synthetic_image(int h, int w, uint64_t seed, float* out) {
    if (h < 1 || w < 1) return fail(CC_ERR_CONFIG, "image dimensions must be positive");
    ccs_make_image(h, w, seed, out);
    return CC_OK;
}

int cc_trainer_create(const float* image, int h, int w, const cc_encoder_config* enc,
                      const cc_decoder_config* dec, int device, cc_trainer** out) {
    (void)device;
    if (h < 1 || w < 1) return fail(CC_ERR_CONFIG, "image dimensions must be positive");
    if (enc->use_soap) return fail(CC_ERR_CONFIG, "the port implements use_soap = false only");
    cc_trainer* T = (cc_trainer*)calloc(1, sizeof(cc_trainer));
    T->H = h;
    T->W = w;
    T->npix = (int64_t)h * w;
    T->enc = *enc;
    snprintf(T->log_path, sizeof(T->log_path), "%s", enc->log_path ? enc->log_path : "");
    T->enc.log_path = NULL;
    const int rc = build(T, dec);
    if (rc != CC_OK) {
        free(T);
        return rc;
    }
    T->img = zalloc(3 * (size_t)T->npix);
    memcpy(T->img, image, sizeof(float) * 3 * (size_t)T->npix);
    *out = T;
    return CC_OK;
}

void cc_trainer_destroy(cc_trainer* T) {
    if (!T) return;
    free(T->img); free(T->y); free(T->yg); free(T->lm); free(T->lv); free(T->th1); free(T->th2);
    free(T->q); free(T->par); free(T->grad); free(T->nm); free(T->nv);
    for (int i = 0; i < T->n_grids; ++i) { free(T->pv[i]); free(T->pg[i]); }
    free(T->z); free(T->dz); free(T->h1); free(T->trunk); free(T->post[0]); free(T->post[1]);
    free(T->xhat); free(T->dx);
    for (int k = 1; k < T->L; ++k)
        for (int j = 0; j < k; ++j) {
            free(T->ups_row[k][j]);
            free(T->ups_col[k][j]);
            if (j > 0) free(T->ups_out[k][j]);
        }
    for (int s = 0; s < NSLOT; ++s) { free(T->snaps[s].y); free(T->snaps[s].p); }
    for (int s = 0; s < NCAND; ++s) {
        free(T->cands[s].y); free(T->cands[s].m); free(T->cands[s].v);
        free(T->cands[s].p); free(T->cands[s].nm); free(T->cands[s].nv);
    }
    free(T->records);
    free(T);
}

int cc_trainer_upload_image(cc_trainer* T, const float* image) {
    memcpy(T->img, image, sizeof(float) * 3 * (size_t)T->npix);
    return CC_OK;
}

int cc_trainer_layout(cc_trainer* T, cc_layout* o) {
    o->height = T->H; o->width = T->W; o->levels = T->L; o->hyper_count = T->hyper;
    o->n_grids = T->n_grids; o->n_latents = T->n_lat; o->n_tensors = T->n_t; o->n_params = T->n_par;
    o->pad = T->P;
    return CC_OK;
}

int cc_trainer_grid_info(cc_trainer* T, int gi, cc_grid_info* o) {
    if (gi < 0 || gi >= T->n_grids) return fail(CC_ERR_CONFIG, "grid index");
    o->level = T->g[gi].level; o->hyper = T->g[gi].hyper; o->rows = T->g[gi].rows;
    o->cols = T->g[gi].cols; o->offset = T->g[gi].off; o->ifce_slot = T->g[gi].slot;
    return CC_OK;
}

int cc_trainer_param_info(cc_trainer* T, int ti, cc_param_info* o) {
    if (ti < 0 || ti >= T->n_t) return fail(CC_ERR_CONFIG, "tensor index");
    memset(o->name, 0, sizeof(o->name));
    snprintf(o->name, sizeof(o->name), "%s", T->t[ti].name);
    o->rows = T->t[ti].rows; o->cols = T->t[ti].cols; o->size = T->t[ti].size; o->offset = T->t[ti].off;
    return CC_OK;
}

#define NEED_LOADED(T) do { if (!(T)->loaded) return fail(CC_ERR_STATE, "no candidate loaded"); } while (0)

int cc_trainer_fresh_candidate(cc_trainer* T, int index) {
    fresh_candidate(T, index);
    return CC_OK;
}

static void cp(float* d, const float* s, size_t n) { if (d && s) memcpy(d, s, sizeof(float) * n); }

int cc_trainer_set_state(cc_trainer* T, const float* lat, const float* par, const float* lm,
                         const float* lv, const int64_t* lt, const float* nm, const float* nv,
                         const int64_t* nt) {
    NEED_LOADED(T);
    const size_t nl = (size_t)T->n_lat, np = (size_t)T->n_par;
    cp(T->y, lat, nl); cp(T->par, par, np); cp(T->lm, lm, nl); cp(T->lv, lv, nl);
    cp(T->nm, nm, np); cp(T->nv, nv, np);
    if (lt) memcpy(T->lat_t, lt, sizeof(int64_t) * (size_t)T->n_grids);
    if (nt) memcpy(T->nn_t, nt, sizeof(int64_t) * (size_t)T->n_t);
    return CC_OK;
}

int cc_trainer_get_state(cc_trainer* T, float* lat, float* par, float* lm, float* lv, int64_t* lt,
                         float* nm, float* nv, int64_t* nt) {
    NEED_LOADED(T);
    const size_t nl = (size_t)T->n_lat, np = (size_t)T->n_par;
    cp(lat, T->y, nl); cp(par, T->par, np); cp(lm, T->lm, nl); cp(lv, T->lv, nl);
    cp(nm, T->nm, np); cp(nv, T->nv, np);
    if (lt) memcpy(lt, T->lat_t, sizeof(int64_t) * (size_t)T->n_grids);
    if (nt) memcpy(nt, T->nn_t, sizeof(int64_t) * (size_t)T->n_t);
    return CC_OK;
}

int cc_trainer_get_grads(cc_trainer* T, float* lg, float* pg) {
    NEED_LOADED(T);
    cp(lg, T->yg, (size_t)T->n_lat);
    cp(pg, T->grad, (size_t)T->n_par);
    return CC_OK;
}

int cc_trainer_get_q(cc_trainer* T, int32_t* q) {
    NEED_LOADED(T);
    memcpy(q, T->q, sizeof(int32_t) * (size_t)T->n_lat);
    return CC_OK;
}

int cc_trainer_get_counters(cc_trainer* T, int64_t* gi, int* sk) {
    if (gi) *gi = T->global_iter;
    if (sk) *sk = T->skipped;
    return CC_OK;
}

int cc_trainer_set_counters(cc_trainer* T, int64_t gi, int sk) {
    T->global_iter = gi;
    T->skipped = sk;
    return CC_OK;
}

int cc_trainer_proxy_iteration(cc_trainer* T, double lr, double temp, double noise, double* cost) {
    NEED_LOADED(T);
    const double c = proxy_iteration(T, lr, temp, noise);
    if (cost) *cost = c;
    return CC_OK;
}

int cc_trainer_enqueue_proxy_iterations(cc_trainer* T, int n, const double* lr, const double* temp,
                                        const double* noise) {
    NEED_LOADED(T);
    free(T->records);
    T->records = (double*)calloc(4 * (size_t)(n > 0 ? n : 1), sizeof(double));
    T->n_records = n;
    for (int i = 0; i < n; ++i) {
        double* r = T->records + 4 * (size_t)i;
        r[0] = proxy_iteration(T, lr[i], temp[i], noise[i]);
        r[1] = T->last_mse;
        r[2] = T->last_bits;
        r[3] = (double)T->global_iter;
    }
    return CC_OK;
}

int cc_trainer_proxy_iterations(cc_trainer* T, int n, const double* lr, const double* temp,
                                const double* noise, double* costs, int* ran) {
    const int rc = cc_trainer_enqueue_proxy_iterations(T, n, lr, temp, noise);
    if (rc != CC_OK) return rc;
    int r = n;
    for (int i = 0; i < n; ++i) {
        if (r == n && !isfinite(T->records[4 * (size_t)i])) r = i + 1;
        if (costs) costs[i] = i < r ? T->records[4 * (size_t)i] : NAN;
    }
    if (ran) *ran = r;
    return CC_OK;
}

int cc_trainer_set_stream(cc_trainer* T, void* s) { (void)T; (void)s; return CC_OK; }
int cc_trainer_synchronize(cc_trainer* T) { (void)T; return CC_OK; }
int cc_trainer_reserve_iterations(cc_trainer* T, int n) { (void)T; (void)n; return CC_OK; }
int cc_trainer_last_records(cc_trainer* T, int n, double* rec) {
    if (n > T->n_records) return fail(CC_ERR_CONFIG, "no such records");
    memcpy(rec, T->records, sizeof(double) * 4 * (size_t)n);
    return CC_OK;
}

int cc_trainer_hardround_iteration(cc_trainer* T, double lr, int best, double* cost) {
    NEED_LOADED(T);
    if (best >= NSLOT) return fail(CC_ERR_CONFIG, "snapshot slot");
    const double c = hardround_iteration(T, lr, best);
    if (cost) *cost = c;
    return CC_OK;
}

int cc_trainer_true_cost(cc_trainer* T, double* cost, double* psnr, double* bpp) {
    NEED_LOADED(T);
    const double c = true_cost(T, psnr, bpp);
    if (cost) *cost = c;
    return CC_OK;
}

int cc_trainer_quantize_all(cc_trainer* T) { NEED_LOADED(T); quantize_all(T); return CC_OK; }
int cc_trainer_load_pads_from_q(cc_trainer* T) { NEED_LOADED(T); load_pads_from_q(T); return CC_OK; }

int cc_trainer_last_terms(cc_trainer* T, double* mse, double* bits) {
    if (mse) *mse = T->last_mse;
    if (bits) *bits = T->last_bits;
    return CC_OK;
}

int cc_trainer_snapshot(cc_trainer* T, int slot, double cost) {
    NEED_LOADED(T);
    if (slot < 0 || slot >= NSLOT) return fail(CC_ERR_CONFIG, "snapshot slot");
    snapshot_take(T, slot, cost);
    return CC_OK;
}

int cc_trainer_snapshot_cost(cc_trainer* T, int slot, double* cost) {
    *cost = (slot >= 0 && slot < NSLOT && T->snaps[slot].valid) ? T->snaps[slot].cost : INFINITY;
    return CC_OK;
}

int cc_trainer_restore(cc_trainer* T, int slot) {
    NEED_LOADED(T);
    if (slot < 0 || slot >= NSLOT || !T->snaps[slot].valid) return fail(CC_ERR_STATE, "empty snapshot slot");
    memcpy(T->y, T->snaps[slot].y, sizeof(float) * (size_t)T->n_lat);
    memcpy(T->par, T->snaps[slot].p, sizeof(float) * (size_t)T->n_par);
    return CC_OK;
}

int cc_trainer_reset_optimizers(cc_trainer* T) { NEED_LOADED(T); reset_optimizers(T); return CC_OK; }

int cc_trainer_take_candidate(cc_trainer* T, int slot, double cost) {
    NEED_LOADED(T);
    if (slot < 0 || slot >= NCAND) return fail(CC_ERR_CONFIG, "candidate slot");
    Cand* c = &T->cands[slot];
    const size_t nl = (size_t)T->n_lat, np = (size_t)T->n_par;
    if (!c->y) {
        c->y = zalloc(nl); c->m = zalloc(nl); c->v = zalloc(nl);
        c->p = zalloc(np); c->nm = zalloc(np); c->nv = zalloc(np);
    }
    cp(c->y, T->y, nl); cp(c->m, T->lm, nl); cp(c->v, T->lv, nl);
    cp(c->p, T->par, np); cp(c->nm, T->nm, np); cp(c->nv, T->nv, np);
    memcpy(c->lat_t, T->lat_t, sizeof(T->lat_t));
    memcpy(c->nn_t, T->nn_t, sizeof(T->nn_t));
    c->cost = cost;
    c->valid = 1;
    T->loaded = 0;
    return CC_OK;
}

int cc_trainer_load_candidate(cc_trainer* T, int slot) {
    if (slot < 0 || slot >= NCAND || !T->cands[slot].valid) return fail(CC_ERR_STATE, "empty candidate slot");
    Cand* c = &T->cands[slot];
    const size_t nl = (size_t)T->n_lat, np = (size_t)T->n_par;
    cp(T->y, c->y, nl); cp(T->lm, c->m, nl); cp(T->lv, c->v, nl);
    cp(T->par, c->p, np); cp(T->nm, c->nm, np); cp(T->nv, c->nv, np);
    memcpy(T->lat_t, c->lat_t, sizeof(T->lat_t));
    memcpy(T->nn_t, c->nn_t, sizeof(T->nn_t));
    T->cur_cost = c->cost;
    c->valid = 0;
    zero_pads(T);
    T->loaded = 1;
    return CC_OK;
}

int cc_trainer_candidate_cost(cc_trainer* T, int slot, double* cost) {
    if (slot < 0 || slot >= NCAND || !T->cands[slot].valid) return fail(CC_ERR_STATE, "empty candidate slot");
    *cost = T->cands[slot].cost;
    return CC_OK;
}

/* warmup (encoder.hpp:315-342) */
typedef struct { int slot; double cost; } CC;
static void sort_cc(CC* a, int n) { /* stable insertion sort by cost */
    for (int i = 1; i < n; ++i) {
        CC x = a[i];
        int j = i - 1;
        while (j >= 0 && a[j].cost > x.cost) { a[j + 1] = a[j]; --j; }
        a[j + 1] = x;
    }
}
static void warmup(cc_trainer* T) {
    const cc_encoder_config* e = &T->enc;
    CC c[NCAND];
    const int nc = e->warmup_candidates < NCAND ? e->warmup_candidates : NCAND;
    for (int i = 0; i < nc; ++i) {
        fresh_candidate(T, i);
        for (int k = 0; k < e->warmup_iters; ++k) proxy_iteration(T, e->lr_start, e->temp_start, e->noise_std_start);
        c[i].slot = i;
        c[i].cost = true_cost(T, NULL, NULL);
        cc_trainer_take_candidate(T, i, c[i].cost);
    }
    sort_cc(c, nc);
    int keep = e->warmup_keep < nc ? e->warmup_keep : nc;
    if (nc <= 1) { cc_trainer_load_candidate(T, c[0].slot); return; }
    for (int i = keep; i < nc; ++i) T->cands[c[i].slot].valid = 0;
    for (int i = 0; i < keep; ++i) {
        cc_trainer_load_candidate(T, c[i].slot);
        for (int k = 0; k < e->warmup_iters; ++k) proxy_iteration(T, e->lr_start, e->temp_start, e->noise_std_start);
        c[i].cost = true_cost(T, NULL, NULL);
        cc_trainer_take_candidate(T, c[i].slot, c[i].cost);
    }
    sort_cc(c, keep);
    for (int i = 1; i < keep; ++i) T->cands[c[i].slot].valid = 0;
    cc_trainer_load_candidate(T, c[0].slot);
}

int cc_trainer_warmup(cc_trainer* T) { warmup(T); return CC_OK; }

static double sched(double a, double b, int cosine, int hor, int it) { /* config.hpp:23-29 */
    if (it <= 0) return a;
    if (it >= hor) return b;
    const double t = (double)it / hor;
    if (!cosine) return a + (b - a) * t;
    return b + (a - b) * (1.0 + cos(3.141592653589793 * t)) * 0.5;
}

static void log_row(FILE* f, cc_trainer* T, double proxy, const double* tc) {
    if (!f) return;
    const double psnr = T->last_mse > 0 ? -10.0 * log10(T->last_mse) : 99.0;
    fprintf(f, "%lld,%g,", (long long)T->global_iter, proxy);
    if (tc) fprintf(f, "%g", *tc);
    fprintf(f, ",%g,%g\n", psnr, T->last_bits / (double)T->npix);
}

int cc_trainer_train(cc_trainer* T, cc_train_stats* st, float* lat, int32_t* q, float* par) {
    /* train (encoder.hpp:349-413) — from a fresh trainer state */
    const clock_t t0 = clock();
    const cc_encoder_config* e = &T->enc;
    T->global_iter = 0;
    T->skipped = 0;
    for (int s = 0; s < NSLOT; ++s) T->snaps[s].valid = 0;
    FILE* lf = T->log_path[0] ? fopen(T->log_path, "w") : NULL;
    if (lf) fprintf(lf, "iter,proxy_cost,true_cost,psnr,bpp\n");
    warmup(T);
    const int hor = e->main_iters - 1 > 1 ? e->main_iters - 1 : 1;
    int restarts = 0;
    double lr_scale = 1.0;
    const int best = 0;
    snapshot_take(T, best, true_cost(T, NULL, NULL));
    for (int it = 0; it < e->main_iters; ++it) {
        const double c = proxy_iteration(T, lr_scale * sched(e->lr_start, e->lr_end, 1, hor, it),
                                         sched(e->temp_start, e->temp_end, 0, hor, it),
                                         sched(e->noise_std_start, e->noise_std_end, 0, hor, it));
        if (!isfinite(c)) {
            if (restarts >= 2) break;
            ++restarts;
            lr_scale *= 0.5;
            cc_trainer_restore(T, best);
            reset_optimizers(T);
            ++T->global_iter;
            continue;
        }
        if ((it + 1) % e->true_cost_interval == 0 || it == e->main_iters - 1) {
            const double tc = true_cost(T, NULL, NULL);
            if (tc < T->snaps[best].cost) snapshot_take(T, best, tc);
            log_row(lf, T, c, &tc);
        } else {
            log_row(lf, T, c, NULL);
        }
    }
    cc_trainer_restore(T, best);
    quantize_all(T);
    load_pads_from_q(T);
    for (int it = 0; it < e->hardround_iters; ++it) {
        const double c = hardround_iteration(T, e->hardround_lr, best);
        if (!isfinite(c)) break;
        log_row(lf, T, c, &c);
    }
    {
        const double tc = true_cost(T, NULL, NULL);
        if (tc < T->snaps[best].cost) snapshot_take(T, best, tc);
    }
    cc_trainer_restore(T, best);
    quantize_all(T);
    if (lf) fclose(lf);
    double psnr = 0, bpp = 0;
    const double tc = true_cost(T, &psnr, &bpp);
    if (st) {
        st->iterations = T->global_iter;
        st->true_cost = tc;
        st->psnr = psnr;
        st->rate_bpp = bpp;
        st->restarts = restarts;
        st->skipped_steps = T->skipped;
        st->seconds = (double)(clock() - t0) / CLOCKS_PER_SEC;
    }
    cp(lat, T->y, (size_t)T->n_lat);
    cp(par, T->par, (size_t)T->n_par);
    if (q) memcpy(q, T->q, sizeof(int32_t) * (size_t)T->n_lat);
    return CC_OK;
}

/* element hooks (same codes as ccref_eval_math) */
int ccport_eval_math(int fn, int n, const float* a, const float* b, const float* c, float* out) {
    for (int i = 0; i < n; ++i) {
        switch (fn) {
            case 0: out[i] = cc_exp(a[i]); break;
            case 1: out[i] = cc_log(a[i]); break;
            case 2: out[i] = cc_tanh(a[i]); break;
            case 3: out[i] = softround_value(a[i], b[i]); break;
            case 4: out[i] = laplace_bits(a[i], b[i], c[i]); break;
            case 5: out[i] = (float)quantize_value(a[i], 255); break;
            case 6: {
                const float inv_t = 1.0f / b[i];
                const float f = floorf(a[i]);
                const float th = cc_tanh((a[i] - f - 0.5f) * inv_t);
                out[i] = fmaf(-th, th, 1.0f) * (1.0f / (b[i] * softround_denom(b[i])));
                break;
            }
            default: return fail(CC_ERR_CONFIG, "unknown math function");
        }
    }
    return CC_OK;
}

int ccport_counter_gauss(uint64_t stream, uint64_t idx0, int n, float* out) {
    for (int i = 0; i < n; ++i) out[i] = counter_gauss(stream, idx0 + (uint64_t)i);
    return CC_OK;
}
