/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference join path (see
 * tj_oracle.h). Written from the reference's behaviour, in the reference's branch form
 * (not the GPU's select form), compiled with -ffp-contract=off so the FP64 arithmetic is
 * the reference's own non-FMA sequence. Brute force wherever the reference uses an index
 * structure whose result is exact (R-tree broad phase, best-first k-NN search).
 */
#include "tj_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- geometry */

typedef struct {
    double x, y, z;
} P3;

static P3 psub(P3 a, P3 b) { P3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static P3 padd(P3 a, P3 b) { P3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static P3 pmul(P3 a, double s) { P3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double pdot(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } /* geom.hpp:24 */
static P3 pcross(P3 a, P3 b) {                                                /* geom.hpp:25-27 */
    P3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static double pnorm2(P3 a) { return pdot(a, a); }
static double pdist(P3 a, P3 b) { return sqrt(pnorm2(psub(a, b))); } /* geom.hpp:29-30 */
static double smin(double a, double b) { return (b < a) ? b : a; }   /* std::min */
static double smax(double a, double b) { return (a < b) ? b : a; }   /* std::max */
static double clamp01(double v) { return smin(smax(v, 0.0), 1.0); }  /* std::clamp */
static P3 pt(const double* c) { P3 r = {c[0], c[1], c[2]}; return r; }

typedef struct {
    P3 v[3];
} Tri;

/* src/geom.cpp:11-16 (initializer-list max keeps the first largest) */
static double mindist_box(const double* a, const double* b) {
    double g[3];
    for (int d = 0; d < 3; ++d) {
        double m = 0.0, p = a[d] - b[3 + d], q = b[d] - a[3 + d];
        if (m < p) m = p;
        if (m < q) m = q;
        g[d] = m;
    }
    return sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
}

/* src/geom.cpp:18-24 */
static double point_segment(P3 p, P3 a, P3 b) {
    P3 d = psub(b, a);
    double dd = pnorm2(d);
    if (dd <= 0.0) return pdist(p, a);
    double t = clamp01(pdot(psub(p, a), d) / dd);
    return pdist(p, padd(a, pmul(d, t)));
}

/* src/geom.cpp:29-35 */
static int degenerate(const Tri* t) {
    P3 ab = psub(t->v[1], t->v[0]), ac = psub(t->v[2], t->v[0]), bc = psub(t->v[2], t->v[1]);
    double s2 = pnorm2(ab);
    if (s2 < pnorm2(ac)) s2 = pnorm2(ac);
    if (s2 < pnorm2(bc)) s2 = pnorm2(bc);
    double n2 = pnorm2(pcross(ab, ac));
    return n2 <= 1e-24 * s2 * s2;
}

/* src/geom.cpp:39-80 (Ericson's Voronoi-region walk, early returns) */
static double point_triangle(P3 p, const Tri* t) {
    if (degenerate(t)) {
        double m = point_segment(p, t->v[0], t->v[1]);
        double m1 = point_segment(p, t->v[1], t->v[2]);
        double m2 = point_segment(p, t->v[2], t->v[0]);
        if (m1 < m) m = m1;
        if (m2 < m) m = m2;
        return m;
    }
    P3 a = t->v[0], b = t->v[1], c = t->v[2];
    P3 ab = psub(b, a), ac = psub(c, a), ap = psub(p, a);
    double d1 = pdot(ab, ap), d2 = pdot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return pdist(p, a);
    P3 bp = psub(p, b);
    double d3 = pdot(ab, bp), d4 = pdot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) return pdist(p, b);
    double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return pdist(p, padd(a, pmul(ab, d1 / (d1 - d3))));
    P3 cp = psub(p, c);
    double d5 = pdot(ab, cp), d6 = pdot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return pdist(p, c);
    double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return pdist(p, padd(a, pmul(ac, d2 / (d2 - d6))));
    double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return pdist(p, padd(b, pmul(psub(c, b), w)));
    }
    double den = 1.0 / (va + vb + vc);
    double v = vb * den, w = vc * den;
    return pdist(p, padd(padd(a, pmul(ab, v)), pmul(ac, w)));
}

/* src/geom.cpp:82-113 */
static double segment_segment(P3 p1, P3 q1, P3 p2, P3 q2) {
    P3 d1 = psub(q1, p1), d2 = psub(q2, p2), r = psub(p1, p2);
    double a = pnorm2(d1), e = pnorm2(d2), f = pdot(d2, r), s = 0.0, t = 0.0;
    if (a <= 0.0 && e <= 0.0) return pdist(p1, p2);
    if (a <= 0.0) {
        t = clamp01(f / e);
    } else {
        double c = pdot(d1, r);
        if (e <= 0.0) {
            s = clamp01(-c / a);
        } else {
            double b = pdot(d1, d2), den = a * e - b * b;
            if (den > 0.0) s = clamp01((b * f - c * e) / den);
            t = (b * s + f) / e;
            if (t < 0.0) {
                t = 0.0;
                s = clamp01(-c / a);
            } else if (t > 1.0) {
                t = 1.0;
                s = clamp01((b - c) / a);
            }
        }
    }
    return pdist(padd(p1, pmul(d1, s)), padd(p2, pmul(d2, t)));
}

/* src/geom.cpp:120-136 */
static int pierces(P3 p, P3 q, const Tri* t) {
    P3 dir = psub(q, p), e1 = psub(t->v[1], t->v[0]), e2 = psub(t->v[2], t->v[0]);
    P3 pv = pcross(dir, e2);
    double det = pdot(e1, pv);
    double scale = sqrt(pnorm2(dir)) * sqrt(pnorm2(e1)) * sqrt(pnorm2(e2));
    if (fabs(det) <= 1e-14 * scale) return 0;
    double inv = 1.0 / det;
    P3 tv = psub(p, t->v[0]);
    double u = pdot(tv, pv) * inv;
    if (u < 0.0 || u > 1.0) return 0;
    P3 qv = pcross(tv, e1);
    double v = pdot(dir, qv) * inv;
    if (v < 0.0 || u + v > 1.0) return 0;
    double tt = pdot(e2, qv) * inv;
    return tt >= 0.0 && tt <= 1.0;
}

/* src/geom.cpp:140-148 */
static int tri_less(const Tri* a, const Tri* b) {
    const double* pa = &a->v[0].x;
    const double* pb = &b->v[0].x;
    for (int i = 0; i < 9; ++i) {
        if (pa[i] < pb[i]) return 1;
        if (pa[i] > pb[i]) return 0;
    }
    return 0;
}

/* src/geom.cpp:152-183 */
static double tri_tri(const Tri* ta, const Tri* tb) {
    const Tri* t1 = tri_less(tb, ta) ? tb : ta;
    const Tri* t2 = tri_less(tb, ta) ? ta : tb;
    double best = INFINITY;
    for (int i = 0; i < 3; ++i) {
        best = smin(best, point_triangle(t1->v[i], t2));
        best = smin(best, point_triangle(t2->v[i], t1));
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            best = smin(best, segment_segment(t1->v[i], t1->v[(i + 1) % 3], t2->v[j], t2->v[(j + 1) % 3]));
    if (best > 0.0) {
        if (!degenerate(t2))
            for (int i = 0; i < 3; ++i)
                if (pierces(t1->v[i], t1->v[(i + 1) % 3], t2)) return 0.0;
        if (!degenerate(t1))
            for (int j = 0; j < 3; ++j)
                if (pierces(t2->v[j], t2->v[(j + 1) % 3], t1)) return 0.0;
    }
    return best;
}

static Tri tri_of(const double* c) {
    Tri t;
    for (int k = 0; k < 3; ++k) t.v[k] = pt(c + 3 * k);
    return t;
}

void ora_tri_tri_batch(uint64_t n, const double* a9, const double* b9, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        Tri a = tri_of(a9 + 9 * i), b = tri_of(b9 + 9 * i);
        out[i] = tri_tri(&a, &b);
    }
}

void ora_mindist_batch(uint64_t n, const double* a6, const double* b6, double* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = mindist_box(a6 + 6 * i, b6 + 6 * i);
}

/* src/refine.cpp:63-84 (t = i * s_len + j, row-major) */
static void refine_one(const Tri* R, const double* rhd, const double* rph, uint32_t rn, const Tri* S,
                       const double* shd, const double* sph, uint32_t sn, double* lb_out, double* ub_out) {
    double lb = INFINITY, ub = INFINITY;
    for (uint32_t i = 0; i < rn; ++i)
        for (uint32_t j = 0; j < sn; ++j) {
            double d = tri_tri(&R[i], &S[j]);
            lb = smin(lb, smax(0.0, d - rph[i] - sph[j]));
            ub = smin(ub, d + rhd[i] + shd[j]);
        }
    *lb_out = lb;
    *ub_out = ub;
}

void ora_refine_batch(uint64_t n_descs, const double* tris9, const double* hd, const double* ph,
                      const uint64_t* r_off, const uint64_t* s_off, const uint32_t* r_len,
                      const uint32_t* s_len, double* vp_lb, double* vp_ub) {
    for (uint64_t d = 0; d < n_descs; ++d) {
        Tri* R = malloc(sizeof(Tri) * (r_len[d] ? r_len[d] : 1));
        Tri* S = malloc(sizeof(Tri) * (s_len[d] ? s_len[d] : 1));
        for (uint32_t i = 0; i < r_len[d]; ++i) R[i] = tri_of(tris9 + 9 * (r_off[d] + i));
        for (uint32_t j = 0; j < s_len[d]; ++j) S[j] = tri_of(tris9 + 9 * (s_off[d] + j));
        refine_one(R, hd + r_off[d], ph + r_off[d], r_len[d], S, hd + s_off[d], ph + s_off[d], s_len[d], &vp_lb[d],
                   &vp_ub[d]);
        free(R);
        free(S);
    }
}

/* ---------------------------------------------------------------- 3DPJ1 reader
 * Container layout per src/index_io.cpp:109-149 (magic, version, lod schedule, objects as
 * length-prefixed bodies). Only the fields the join reads are kept. */

typedef struct {
    uint64_t nf;        /* facets of the level mesh */
    Tri* tris;          /* per facet, level mesh */
    double *hd, *ph;    /* per facet */
    uint64_t* voff;     /* [nvox+1] into vid */
    uint32_t* vid;      /* facet ids per voxel, ascending */
} OLevel;

typedef struct {
    double mbb[6], anchor[3];
    uint32_t nvox;
    double *vbox, *vanc;
    OLevel* lv;
} OObj;

typedef struct {
    uint32_t nl;
    int32_t* levels;
    uint64_t n;
    OObj* o;
} ODs;

typedef struct {
    const unsigned char* p;
    size_t n, at;
    int bad;
} Rd;

static void rd_take(Rd* r, void* dst, size_t k) {
    if (r->bad || r->at + k > r->n) {
        r->bad = 1;
        memset(dst, 0, k);
        return;
    }
    memcpy(dst, r->p + r->at, k);
    r->at += k;
}
static uint32_t rd_u32(Rd* r) { uint32_t v; rd_take(r, &v, 4); return v; }
static uint64_t rd_u64(Rd* r) { uint64_t v; rd_take(r, &v, 8); return v; }
static double rd_f64(Rd* r) { double v; rd_take(r, &v, 8); return v; }

static void ds_free(ODs* d) {
    if (!d->o) return;
    for (uint64_t i = 0; i < d->n; ++i) {
        OObj* o = &d->o[i];
        if (o->lv)
            for (uint32_t l = 0; l < d->nl; ++l) {
                free(o->lv[l].tris);
                free(o->lv[l].hd);
                free(o->lv[l].ph);
                free(o->lv[l].voff);
                free(o->lv[l].vid);
            }
        free(o->lv);
        free(o->vbox);
        free(o->vanc);
    }
    free(d->o);
    free(d->levels);
    memset(d, 0, sizeof(*d));
}

static int ds_load(const char* path, ODs* d) {
    memset(d, 0, sizeof(*d));
    FILE* f = fopen(path, "rb");
    if (!f) return 0;
    fseek(f, 0, SEEK_END);
    long len = ftell(f);
    fseek(f, 0, SEEK_SET);
    unsigned char* buf = malloc(len > 0 ? (size_t)len : 1);
    size_t got = fread(buf, 1, (size_t)len, f);
    fclose(f);
    Rd r = {buf, got, 0, 0};
    char magic[5];
    rd_take(&r, magic, 5);
    if (memcmp(magic, "3DPJ1", 5) != 0 || rd_u32(&r) != 1) r.bad = 1;
    d->nl = rd_u32(&r);
    d->levels = calloc(d->nl ? d->nl : 1, sizeof(int32_t));
    for (uint32_t i = 0; i < d->nl; ++i) d->levels[i] = (int32_t)rd_u32(&r);
    d->n = rd_u64(&r);
    if (r.bad) { free(buf); return 0; }
    d->o = calloc(d->n ? d->n : 1, sizeof(OObj));
    for (uint64_t oi = 0; oi < d->n && !r.bad; ++oi) {
        OObj* o = &d->o[oi];
        rd_u64(&r); /* body length */
        rd_u32(&r); /* id */
        for (int k = 0; k < 6; ++k) o->mbb[k] = rd_f64(&r);
        for (int k = 0; k < 3; ++k) o->anchor[k] = rd_f64(&r);
        uint32_t nlv = rd_u32(&r);
        if (nlv != d->nl) { r.bad = 1; break; }
        o->lv = calloc(nlv, sizeof(OLevel));
        for (uint32_t l = 0; l < nlv && !r.bad; ++l) {
            OLevel* L = &o->lv[l];
            rd_u32(&r);
            unsigned char cl;
            rd_take(&r, &cl, 1);
            uint64_t nv = rd_u64(&r);
            double* v = malloc(24 * (nv ? nv : 1));
            for (uint64_t i = 0; i < 3 * nv; ++i) v[i] = rd_f64(&r);
            uint64_t nf = rd_u64(&r);
            L->nf = nf;
            L->tris = malloc(sizeof(Tri) * (nf ? nf : 1));
            for (uint64_t i = 0; i < nf; ++i)
                for (int k = 0; k < 3; ++k) {
                    uint32_t vi = rd_u32(&r);
                    if (vi >= nv) { r.bad = 1; vi = 0; }
                    L->tris[i].v[k] = pt(v + 3 * (uint64_t)vi);
                }
            free(v);
            L->hd = malloc(8 * (nf ? nf : 1));
            L->ph = malloc(8 * (nf ? nf : 1));
            for (uint64_t i = 0; i < nf; ++i) L->hd[i] = rd_f64(&r);
            for (uint64_t i = 0; i < nf; ++i) L->ph[i] = rd_f64(&r);
            uint64_t na = rd_u64(&r);
            for (uint64_t i = 0; i < na; ++i) rd_u32(&r); /* ancestor map: not on the join path */
        }
        o->nvox = rd_u32(&r);
        rd_u32(&r); /* reassigned */
        o->vbox = malloc(48 * (o->nvox ? o->nvox : 1));
        o->vanc = malloc(24 * (o->nvox ? o->nvox : 1));
        for (uint32_t v = 0; v < o->nvox; ++v) {
            for (int k = 0; k < 6; ++k) o->vbox[6 * v + k] = rd_f64(&r);
            for (int k = 0; k < 3; ++k) o->vanc[3 * v + k] = rd_f64(&r);
        }
        for (uint32_t l = 0; l < nlv && !r.bad; ++l) {
            OLevel* L = &o->lv[l];
            L->voff = calloc(o->nvox + 1, sizeof(uint64_t));
            size_t cap = 64, used = 0;
            L->vid = malloc(4 * cap);
            for (uint32_t v = 0; v < o->nvox; ++v) {
                uint64_t c = rd_u64(&r);
                if (r.bad) break;
                for (uint64_t i = 0; i < c; ++i) {
                    if (used == cap) { cap *= 2; L->vid = realloc(L->vid, 4 * cap); }
                    L->vid[used++] = rd_u32(&r);
                }
                L->voff[v + 1] = used;
            }
        }
    }
    int ok = !r.bad && r.at == r.n;
    free(buf);
    if (!ok) ds_free(d);
    return ok;
}

/* ---------------------------------------------------------------- join */

enum { UND = 0, CONF = 1, REM = 2 };
enum { ST_NONE = -3, ST_MBB = -2, ST_VOXEL = -1 };

typedef struct {
    uint64_t n;
    uint32_t *r, *s;
    double *lb, *ub;
    uint8_t* st;
    int16_t* at;
    uint64_t* r2op;
    uint32_t* nconf;
} Cands;

typedef struct {
    uint32_t op, vr, vs;
} Avp;

typedef struct {
    ora_result* out;
    int failed;
} Ctx;

static void fail(Ctx* c, int status, const char* msg) {
    if (c->failed) return;
    c->failed = 1;
    c->out->status = status;
    snprintf(c->out->error, sizeof(c->out->error), "%s", msg);
}

/* src/filter.cpp:22-32 */
static void intersect(Ctx* c, double* lb, double* ub, double nlb, double nub) {
    *lb = smax(*lb, nlb);
    *ub = smin(*ub, nub);
    if (*lb > *ub) {
        if (*lb - *ub > 1e-9) fail(c, 2, "bound crossing");
        double mid = 0.5 * (*lb + *ub);
        *lb = *ub = mid;
    }
}

/* src/filter.cpp:241-263 */
static void prune_op(Cands* k, uint64_t op, double tau, int16_t code) {
    if (k->st[op] != UND) return;
    if (k->ub[op] <= tau) {
        k->st[op] = CONF;
        k->at[op] = code;
        ++k->nconf[k->r[op]];
    } else if (k->lb[op] > tau) {
        k->st[op] = REM;
        k->at[op] = code;
    }
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* src/knn.cpp:19-91: global snapshot rounds until no decision changes. */
static void knn_fixpoint(Ctx* c, Cands* k, uint32_t nq, uint32_t kk, int16_t code) {
    uint8_t* delta = calloc(k->n ? k->n : 1, 1);
    for (;;) {
        uint64_t nd = 0;
        for (uint32_t r = 0; r < nq; ++r) {
            uint64_t b = k->r2op[r], e = k->r2op[r + 1];
            int64_t u = 0;
            for (uint64_t m = b; m < e; ++m) u += k->st[m] == UND;
            if (u == 0) continue;
            int64_t kleft = (int64_t)kk - (int64_t)k->nconf[r];
            if (kleft < 0) { fail(c, 2, "knn_prune_round: confirmed count exceeds k"); break; }
            for (uint64_t m = b; m < e; ++m) {
                if (k->st[m] != UND) continue;
                int64_t farther = 0, closer = 0;
                for (uint64_t n = b; n < e; ++n) {
                    if (k->st[n] != UND) continue;
                    farther += k->lb[n] > k->ub[m];
                    closer += k->ub[n] < k->lb[m];
                }
                if ((u - 1) - farther < kleft) { delta[m] = CONF; ++nd; }
                else if (closer >= kleft) { delta[m] = REM; ++nd; }
            }
        }
        if (nd == 0 || c->failed) break;
        for (uint64_t m = 0; m < k->n; ++m) {
            if (!delta[m]) continue;
            k->st[m] = delta[m];
            k->at[m] = code;
            if (delta[m] == CONF && ++k->nconf[k->r[m]] > kk) fail(c, 2, "knn_apply_deltas: confirmed count exceeds k");
            delta[m] = 0;
        }
    }
    free(delta);
}

static int level_slot(const ODs* d, uint32_t level) {
    for (uint32_t i = 0; i < d->nl; ++i)
        if (d->levels[i] == (int32_t)level) return (int)i;
    return -1;
}

typedef struct {
    double key;
    uint32_t s;
    uint64_t op;
    double lb2;
} SortKey;

static int cmp_finalize(const void* a, const void* b) { /* (lb, s) */
    const SortKey *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return (x->s > y->s) - (x->s < y->s);
}
static int cmp_records(const void* a, const void* b) { /* (ub, lb, s) */
    const SortKey *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->lb2 != y->lb2) return x->lb2 < y->lb2 ? -1 : 1;
    return (x->s > y->s) - (x->s < y->s);
}

void ora_join_files(const char* r_path, const char* s_path, int type, double tau, uint32_t kk,
                    const uint32_t* lods, uint32_t n_lods, ora_result* out) {
    ora_join_files_ex(r_path, s_path, type, tau, kk, lods, n_lods, 0, out);
}

void ora_join_files_ex(const char* r_path, const char* s_path, int type, double tau, uint32_t kk,
                       const uint32_t* lods, uint32_t n_lods, int exact, ora_result* out) {
    memset(out, 0, sizeof(*out));
    Ctx c = {out, 0};
    const int knn = type == 2;
    if (type == 1) tau = 0.0;
    ODs R, Sown, *S = &R;
    if (!ds_load(r_path, &R)) { fail(&c, 3, "cannot read R index"); return; }
    int self = !s_path || !*s_path || strcmp(s_path, r_path) == 0;
    if (!self) {
        if (!ds_load(s_path, &Sown)) { ds_free(&R); fail(&c, 3, "cannot read S index"); return; }
        S = &Sown;
    }
    const uint32_t nq = (uint32_t)R.n, ns = (uint32_t)S->n;
    Cands k;
    memset(&k, 0, sizeof(k));
    k.r2op = calloc((size_t)nq + 1, 8);
    k.nconf = calloc(nq ? nq : 1, 4);
    /* ---- MBB stage: brute-force restatement of the exact R-tree result ---- */
    size_t cap = 1024;
    k.r = malloc(4 * cap); k.s = malloc(4 * cap); k.lb = malloc(8 * cap); k.ub = malloc(8 * cap);
    double* ad = malloc(8 * (ns ? ns : 1));
    for (uint32_t r = 0; r < nq; ++r) {
        double thr = tau;
        if (knn) { /* u_k(r): k-th smallest anchor distance over all of S */
            for (uint32_t s = 0; s < ns; ++s) ad[s] = pdist(pt(R.o[r].anchor), pt(S->o[s].anchor));
            qsort(ad, ns, 8, cmp_double);
            thr = ns >= kk ? ad[kk - 1] : INFINITY;
        }
        k.r2op[r] = k.n;
        for (uint32_t s = 0; s < ns; ++s) {
            double lb = mindist_box(R.o[r].mbb, S->o[s].mbb);
            if (!(lb <= thr)) continue;
            if (k.n == cap) {
                cap *= 2;
                k.r = realloc(k.r, 4 * cap); k.s = realloc(k.s, 4 * cap);
                k.lb = realloc(k.lb, 8 * cap); k.ub = realloc(k.ub, 8 * cap);
            }
            k.r[k.n] = r; k.s[k.n] = s; k.lb[k.n] = lb;
            k.ub[k.n] = pdist(pt(R.o[r].anchor), pt(S->o[s].anchor));
            ++k.n;
        }
    }
    k.r2op[nq] = k.n;
    free(ad);
    k.st = calloc(k.n ? k.n : 1, 1);
    k.at = malloc(2 * (k.n ? k.n : 1));
    for (uint64_t op = 0; op < k.n; ++op) {
        k.at[op] = ST_NONE;
        if (!knn && k.ub[op] <= tau) { k.st[op] = CONF; k.at[op] = ST_MBB; ++k.nconf[k.r[op]]; }
    }
    if (knn) knn_fixpoint(&c, &k, nq, kk, ST_MBB);

    /* ---- voxel-pair stage (src/filter.cpp:199-315; chunking is result-invariant) ---- */
    uint64_t vpg = 0, vpp = 0, na = 0, acap = 1024;
    Avp* act = malloc(sizeof(Avp) * acap);
    for (uint64_t op = 0; op < k.n && !c.failed; ++op) {
        if (k.st[op] != UND) continue;
        const OObj *ro = &R.o[k.r[op]], *so = &S->o[k.s[op]];
        uint64_t total = (uint64_t)ro->nvox * so->nvox;
        double mlb = INFINITY, mub = INFINITY;
        for (uint64_t t = 0; t < total; ++t) {
            uint64_t i = t / so->nvox, j = t % so->nvox;
            mlb = smin(mlb, mindist_box(ro->vbox + 6 * i, so->vbox + 6 * j));
            mub = smin(mub, pdist(pt(ro->vanc + 3 * i), pt(so->vanc + 3 * j)));
        }
        intersect(&c, &k.lb[op], &k.ub[op], mlb, mub);
        if (!knn) prune_op(&k, op, tau, ST_VOXEL);
        vpg += total;
        if (k.st[op] != UND) continue;
        uint64_t surv = 0;
        for (uint64_t t = 0; t < total; ++t) {
            uint64_t i = t / so->nvox, j = t % so->nvox;
            if (!(mindist_box(ro->vbox + 6 * i, so->vbox + 6 * j) <= k.ub[op])) continue;
            if (na == acap) { acap *= 2; act = realloc(act, sizeof(Avp) * acap); }
            act[na].op = (uint32_t)op; act[na].vr = (uint32_t)i; act[na].vs = (uint32_t)j;
            ++na;
            ++surv;
        }
        vpp += total - surv;
    }
    if (knn && !c.failed) knn_fixpoint(&c, &k, nq, kk, ST_VOXEL);

    /* ---- refinement (src/refine.cpp:263-314) ---- */
    uint64_t lvps[20] = {0}, lfp[20] = {0};
    for (uint32_t li = 0; li < n_lods && !c.failed; ++li) {
        int sr = level_slot(&R, lods[li]), ss = level_slot(S, lods[li]);
        if (sr < 0 || ss < 0) { fail(&c, 2, "refine: level is not in the dataset's lod schedule"); break; }
    }
    /* drop voxel pairs of ops decided by the voxel-stage k-NN round */
    uint64_t w = 0;
    for (uint64_t i = 0; i < na; ++i)
        if (k.st[act[i].op] == UND) act[w++] = act[i];
    na = w;
    double *olb = malloc(8 * (k.n ? k.n : 1)), *oub = malloc(8 * (k.n ? k.n : 1));
    for (uint32_t li = 0; li < n_lods && !c.failed; ++li) {
        if (na == 0) break;
        int sr = level_slot(&R, lods[li]), ss = level_slot(S, lods[li]);
        for (uint64_t op = 0; op < k.n; ++op) olb[op] = oub[op] = INFINITY;
        lvps[li] = na;
        for (uint64_t i = 0; i < na; ++i) {
            const Avp* a = &act[i];
            const OLevel *Lr = &R.o[k.r[a->op]].lv[sr], *Ls = &S->o[k.s[a->op]].lv[ss];
            uint64_t rb = Lr->voff[a->vr], re = Lr->voff[a->vr + 1], sb = Ls->voff[a->vs], se = Ls->voff[a->vs + 1];
            lfp[li] += (re - rb) * (se - sb);
            double lb = INFINITY, ub = INFINITY;
            for (uint64_t x = rb; x < re; ++x)
                for (uint64_t y = sb; y < se; ++y) {
                    uint32_t fi = Lr->vid[x], fj = Ls->vid[y];
                    double d = tri_tri(&Lr->tris[fi], &Ls->tris[fj]);
                    lb = smin(lb, smax(0.0, d - Lr->ph[fi] - Ls->ph[fj]));
                    ub = smin(ub, d + Lr->hd[fi] + Ls->hd[fj]);
                }
            olb[a->op] = smin(olb[a->op], lb);
            oub[a->op] = smin(oub[a->op], ub);
        }
        /* aggregate_object_bounds (src/refine.cpp:86-122), then prune / k-NN rounds */
        for (uint64_t op = 0; op < k.n; ++op) {
            if (k.st[op] != UND || isinf(olb[op])) continue;
            intersect(&c, &k.lb[op], &k.ub[op], olb[op], oub[op]);
        }
        if (knn) knn_fixpoint(&c, &k, nq, kk, (int16_t)lods[li]);
        else
            for (uint64_t op = 0; op < k.n; ++op) prune_op(&k, op, tau, (int16_t)lods[li]);
        w = 0;
        for (uint64_t i = 0; i < na; ++i)
            if (k.st[act[i].op] == UND) act[w++] = act[i];
        na = w;
    }
    free(olb);
    free(oub);
    free(act);
    if (!c.failed) {
        if (knn) { /* knn_finalize (src/knn.cpp:93-118) */
            SortKey* sk = malloc(sizeof(SortKey) * (k.n ? k.n : 1));
            for (uint32_t r = 0; r < nq; ++r) {
                size_t m = 0;
                for (uint64_t op = k.r2op[r]; op < k.r2op[r + 1]; ++op)
                    if (k.st[op] == UND) { sk[m].key = k.lb[op]; sk[m].s = k.s[op]; sk[m].op = op; ++m; }
                qsort(sk, m, sizeof(SortKey), cmp_finalize);
                uint32_t kl = kk > k.nconf[r] ? kk - k.nconf[r] : 0;
                for (size_t i = 0; i < m; ++i) {
                    if (kl > 0) { k.st[sk[i].op] = CONF; ++k.nconf[r]; --kl; }
                    else k.st[sk[i].op] = REM;
                    k.at[sk[i].op] = 100;
                }
            }
            free(sk);
        } else {
            for (uint64_t op = 0; op < k.n; ++op)
                if (k.st[op] == UND) { fail(&c, 2, "refine_loop: candidates left undecided after the exact level"); break; }
        }
    }
    if (!c.failed && exact) {
        /* --exact (src/engine.cpp:96-118, :159): each confirmed interval becomes [d, d], d the
           minimum tri_tri_distance over all facet pairs of the two level-100 meshes (the
           reference's TriBvh::pair_distance, src/bvh.cpp:114-154, is that minimum; here by
           brute force) */
        const int sr = level_slot(&R, 100), ss = level_slot(S, 100);
        for (uint64_t op = 0; op < k.n && sr >= 0 && ss >= 0; ++op) {
            if (k.st[op] != CONF) continue;
            const OLevel* a = &R.o[k.r[op]].lv[sr];
            const OLevel* b = &S->o[k.s[op]].lv[ss];
            double d = INFINITY;
            for (uint64_t i = 0; i < a->nf && d != 0.0; ++i)
                for (uint64_t j = 0; j < b->nf; ++j) {
                    d = smin(d, tri_tri(&a->tris[i], &b->tris[j]));
                    if (d == 0.0) break;
                }
            k.lb[op] = k.ub[op] = d;
        }
    }
    if (!c.failed) {
        /* records (src/engine.cpp:161-185) */
        out->records = malloc(sizeof(ora_record) * (k.n ? k.n : 1));
        SortKey* sk = malloc(sizeof(SortKey) * (k.n ? k.n : 1));
        for (uint32_t r = 0; r < nq; ++r) {
            size_t m = 0;
            for (uint64_t op = k.r2op[r]; op < k.r2op[r + 1]; ++op)
                if (k.st[op] == CONF) {
                    sk[m].key = knn ? k.ub[op] : (double)m;
                    sk[m].lb2 = k.lb[op];
                    sk[m].s = k.s[op];
                    sk[m].op = op;
                    ++m;
                }
            if (knn) qsort(sk, m, sizeof(SortKey), cmp_records);
            for (size_t i = 0; i < m; ++i) {
                ora_record* rec = &out->records[out->n_records++];
                uint64_t op = sk[i].op;
                rec->r = r; rec->s = k.s[op]; rec->lb = k.lb[op]; rec->ub = k.ub[op];
                rec->stage = k.at[op]; rec->rank = knn ? (uint32_t)(i + 1) : 0;
            }
        }
        free(sk);
        /* stage counters (src/engine.cpp:188-236) */
        uint64_t all = (uint64_t)nq * ns, flowing = all;
        int16_t codes[20];
        uint32_t nst = 0;
        codes[nst++] = ST_MBB;
        codes[nst++] = ST_VOXEL;
        for (uint32_t li = 0; li < n_lods && nst < 20; ++li) codes[nst++] = (int16_t)lods[li];
        for (uint32_t si = 0; si < nst; ++si) {
            ora_stage* st = &out->stages[si];
            st->code = codes[si];
            for (uint64_t op = 0; op < k.n; ++op) {
                if (k.at[op] != codes[si]) continue;
                if (k.st[op] == CONF) ++st->confirmed;
                else if (k.st[op] == REM) ++st->removed;
            }
            if (codes[si] == ST_MBB) st->removed += all - k.n;
            if (codes[si] == ST_VOXEL) { st->vp_generated = vpg; st->vp_pruned = vpp; }
            if (si >= 2) { st->vp_generated = lvps[si - 2]; st->facet_pairs = lfp[si - 2]; }
            st->pairs_in = flowing;
            st->pairs_out = flowing - st->confirmed - st->removed;
            flowing = st->pairs_out;
        }
        out->n_stages = nst;
    }
    free(k.r); free(k.s); free(k.lb); free(k.ub); free(k.st); free(k.at); free(k.r2op); free(k.nconf);
    ds_free(&R);
    if (!self) ds_free(&Sown);
}

void ora_result_free(ora_result* r) {
    free(r->records);
    r->records = NULL;
    r->n_records = 0;
}
