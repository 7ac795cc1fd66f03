/*
 * styleblit_oracle.c -- CPU ORACLE for StyleBlit (arXiv 1807.03249).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  Never linked into or called by the product
 * (paper_1807_03249_b200/).  Shares no source with it.
 *
 * Plain C99, fp64 where the paper writes a real-valued formula, written in the paper's
 * order and notation (Alg. 2; voting, lines 412-421).  No
 * blocking, no tables, no reordering: it is meant to be checked against the paper by eye.
 * Readings R1..R27 of ambiguous passages are listed in DESIGN.md.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): SURVEY App. A hash vectors, SPEC's
 * worked SeedPoint/NearestSeed examples, closed-form NearestSeed on the zero-jitter
 * grid, an independent numpy brute-force LUT, the identity / translation / t=0
 * (Lit Sphere) closed forms, the seed-pixel property, the error bound, monotonicity
 * in t, and a hand-computed vote.
 */
#include "styleblit_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

const char* or_version(void) { return "styleblit-oracle 1.0 (C99, fp64)"; }

/* ------------------------------------------------------------------------------------ */
/* R5: RandomJitterTable[b] realised as a stateless hash.  */
/* ------------------------------------------------------------------------------------ */
uint32_t or_lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

uint32_t or_cell_hash(int32_t bx, int32_t by, int32_t l, uint32_t seed) {
    uint32_t c_l = or_lowbias32((uint32_t)l ^ or_lowbias32(seed));
    return or_lowbias32((uint32_t)bx ^ or_lowbias32((uint32_t)by ^ c_l));
}

/* j in [0,1)^2: the low 16 bits of the hash give j_x, the high 16 bits give j_y. */
void or_jitter(int32_t bx, int32_t by, int32_t l, uint32_t seed, int32_t zero_jitter,
               double* jx, double* jy) {
    if (zero_jitter) { *jx = 0.0; *jy = 0.0; return; }
    uint32_t k = or_cell_hash(bx, by, l, seed);
    *jx = (double)(k & 0xFFFFu) / 65536.0;
    *jy = (double)(k >> 16) / 65536.0;
}

/* floor(p/h) toward -infinity (R6). */
static int32_t floor_div(int32_t p, int32_t h) {
    return (int32_t)floor((double)p / (double)h);
}

/* Alg. 2, SeedPoint:
 *   b = floor(p/h);  j = RandomJitterTable[b];  return floor(h * (b + j)).      */
void or_seed_point_j(int32_t px, int32_t py, int32_t h, double jx, double jy,
                     int32_t* sx, int32_t* sy) {
    int32_t bx = floor_div(px, h), by = floor_div(py, h);
    *sx = (int32_t)floor((double)h * ((double)bx + jx));
    *sy = (int32_t)floor((double)h * ((double)by + jy));
}

void or_seed_point(int32_t px, int32_t py, int32_t l, uint32_t seed, int32_t zero_jitter,
                   int32_t* sx, int32_t* sy) {
    int32_t h = 1 << l;
    int32_t bx = floor_div(px, h), by = floor_div(py, h);
    double jx, jy;
    or_jitter(bx, by, l, seed, zero_jitter, &jx, &jy);
    or_seed_point_j(px, py, h, jx, jy, sx, sy);
}

/* Alg. 2, NearestSeed.  x outer, y inner, keep the first strictly
 * smaller d = ||s - p|| (Euclidean, in fp64; exact ordering for integer offsets, R1, R7). */
void or_nearest_seed(int32_t px, int32_t py, int32_t l, uint32_t seed, int32_t zero_jitter,
                     int32_t* qx, int32_t* qy) {
    int32_t h = 1 << l;
    double d_star = INFINITY;
    int32_t best_x = 0, best_y = 0;
    for (int32_t x = -1; x <= 1; ++x) {
        for (int32_t y = -1; y <= 1; ++y) {
            int32_t sx, sy;
            or_seed_point(px + h * x, py + h * y, l, seed, zero_jitter, &sx, &sy);
            double dx = (double)sx - (double)px, dy = (double)sy - (double)py;
            double d = sqrt(dx * dx + dy * dy);
            if (d < d_star) { best_x = sx; best_y = sy; d_star = d; }
        }
    }
    *qx = best_x;
    *qy = best_y;
}

/* ------------------------------------------------------------------------------------ */
/* Guide look-up table ("simple look-up table", Alg. 2).       */
/* ------------------------------------------------------------------------------------ */
uint32_t or_lut_entry(const uint8_t* gs, int32_t ws, int32_t hs, int32_t g0, int32_t g1) {
    /* u* = argmin_u ||(g0,g1) - G_S[u].(c0,c1)||, scanning u in row-major order and keeping
     * the first strict minimum (R10).  The squared norm has the same argmin.           */
    int64_t best = -1;
    uint32_t best_u = 0;
    for (int32_t y = 0; y < hs; ++y) {
        for (int32_t x = 0; x < ws; ++x) {
            const uint8_t* g = gs + 4 * ((int64_t)y * ws + x);
            int64_t d0 = (int64_t)g0 - g[0], d1 = (int64_t)g1 - g[1];
            int64_t d = d0 * d0 + d1 * d1;
            if (best < 0 || d < best) { best = d; best_u = (uint32_t)x | ((uint32_t)y << 16); }
        }
    }
    return best_u;
}

/* Exact guide search over three channels (the look-up "or a tree search";
 * SURVEY 8(f) #3): u* = argmin_u ||(g0,g1,g2) - G_S[u].(c0,c1,c2)||, row-major scan, first
 * strict minimum (the tie rule of R10).  Reading R26.                                     */
uint32_t or_lut3_entry(const uint8_t* gs, int32_t ws, int32_t hs, int32_t g0, int32_t g1, int32_t g2) {
    int64_t best = -1;
    uint32_t best_u = 0;
    for (int32_t y = 0; y < hs; ++y) {
        for (int32_t x = 0; x < ws; ++x) {
            const uint8_t* g = gs + 4 * ((int64_t)y * ws + x);
            int64_t d0 = (int64_t)g0 - g[0], d1 = (int64_t)g1 - g[1], d2 = (int64_t)g2 - g[2];
            int64_t d = d0 * d0 + d1 * d1 + d2 * d2;
            if (best < 0 || d < best) { best = d; best_u = (uint32_t)x | ((uint32_t)y << 16); }
        }
    }
    return best_u;
}

typedef struct {
    const uint8_t* gs; int32_t ws, hs; const uint32_t* keys; uint32_t* out; int64_t b, e;
} lut3_job;

static void* lut3_worker(void* arg) {
    lut3_job* j = (lut3_job*)arg;
    for (int64_t i = j->b; i < j->e; ++i) {
        uint32_t k = j->keys[i];
        j->out[i] = or_lut3_entry(j->gs, j->ws, j->hs, k & 0xFF, (k >> 8) & 0xFF, (k >> 16) & 0xFF);
    }
    return NULL;
}

/* or_lut3_entry for a list of keys k = g0 | g1<<8 | g2<<16 (threads split the list). */
void or_lut3_entries(const uint8_t* gs, int32_t ws, int32_t hs, const uint32_t* keys, int64_t n,
                     uint32_t* out, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    lut3_job jobs[256];
    for (int32_t i = 0; i < nthreads; ++i) {
        lut3_job j = {gs, ws, hs, keys, out, n * i / nthreads, n * (i + 1) / nthreads};
        jobs[i] = j;
    }
    if (nthreads == 1) { lut3_worker(&jobs[0]); return; }
    for (int32_t i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, lut3_worker, &jobs[i]);
    for (int32_t i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

typedef struct {
    const uint8_t* gs; int32_t ws, hs; uint32_t* lut; int32_t k_begin, k_end;
} lut_job;

static void* lut_worker(void* arg) {
    lut_job* j = (lut_job*)arg;
    for (int32_t k = j->k_begin; k < j->k_end; ++k)
        j->lut[k] = or_lut_entry(j->gs, j->ws, j->hs, k & 0xFF, k >> 8);
    return NULL;
}

void or_build_lut(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    lut_job jobs[256];
    for (int32_t i = 0; i < nthreads; ++i) {
        jobs[i].gs = gs; jobs[i].ws = ws; jobs[i].hs = hs; jobs[i].lut = lut;
        jobs[i].k_begin = (int32_t)((int64_t)65536 * i / nthreads);
        jobs[i].k_end = (int32_t)((int64_t)65536 * (i + 1) / nthreads);
    }
    if (nthreads == 1) { lut_worker(&jobs[0]); return; }
    for (int32_t i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, lut_worker, &jobs[i]);
    for (int32_t i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------------------------ */
/* Alg. 2, ParallelStyleBlit.                                         */
/* ------------------------------------------------------------------------------------ */
static int32_t clampi(int32_t v, int32_t lo, int32_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* u* for a guide value: the table entry of channels 0 and 1 (R11), or with lut_rgb the exact
 * three-channel search (R26), evaluated directly. */
static uint32_t lut_at(const or_params* prm, const uint32_t* lut, const uint8_t* gs, int32_t ws, int32_t hs,
                       const uint8_t* g) {
    if (prm->lut_rgb) return or_lut3_entry(gs, ws, hs, g[0], g[1], g[2]);
    return lut[(uint32_t)g[0] | ((uint32_t)g[1] << 8)];
}

void or_stylize_pixel(const or_params* prm, const uint8_t* gs, int32_t ws, int32_t hs,
                      const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                      int32_t px, int32_t py, uint32_t* coord, uint8_t* level) {
    const uint8_t* gt_p = gt + 4 * ((int64_t)py * wt + px);
    for (int32_t l = prm->L; l >= 1; --l) {                               /* line 380 */
        int32_t qx, qy;
        or_nearest_seed(px, py, l, prm->seed, prm->zero_jitter, &qx, &qy); /* line 382 */
        qx = clampi(qx, 0, wt - 1);                                        /* R8 */
        qy = clampi(qy, 0, ht - 1);
        uint32_t u = lut_at(prm, lut, gs, ws, hs, gt + 4 * ((int64_t)qy * wt + qx)); /* line 383 */
        int32_t ux = (int32_t)(u & 0xFFFFu), uy = (int32_t)(u >> 16);
        int32_t sx = ux + (px - qx), sy = uy + (py - qy);                  /* u* + (p - q_l) */
        if (sx < 0 || sx >= ws || sy < 0 || sy >= hs) continue;           /* R9 */
        const uint8_t* gs_s = gs + 4 * ((int64_t)sy * ws + sx);
        /* segmentation guide: a chunk never crosses a label boundary */
        if (prm->label_channel >= 0 && gt_p[prm->label_channel] != gs_s[prm->label_channel]) continue;
        double e2 = 0.0;                                                   /* line 384, R1 */
        for (int32_t c = 0; c < prm->C; ++c) {
            if (c == prm->label_channel) continue;
            double d = (double)gt_p[c] - (double)gs_s[c];
            e2 += (double)prm->w[c] * d * d;                               /* weighted channels */
        }
        double e = sqrt(e2);
        if (e < prm->t) {                                                  /* line 385, R3 */
            *coord = (uint32_t)sx | ((uint32_t)sy << 16);                  /* line 387 */
            *level = (uint8_t)l;
            return;                                                        /* line 388 */
        }
    }
    *coord = lut_at(prm, lut, gs, ws, hs, gt_p);                           /* R12 */
    *level = 0;
}

typedef struct {
    const or_params* prm; const uint8_t* cs; const uint8_t* gs; int32_t ws, hs;
    const uint32_t* lut; const uint8_t* gt; int32_t wt, ht;
    uint8_t* ct; uint32_t* coords; uint8_t* level; int32_t y_begin, y_end;
} sty_job;

static void* sty_worker(void* arg) {
    sty_job* j = (sty_job*)arg;
    for (int32_t py = j->y_begin; py < j->y_end; ++py) {
        for (int32_t px = 0; px < j->wt; ++px) {
            int64_t i = (int64_t)py * j->wt + px;
            uint32_t c; uint8_t lv;
            or_stylize_pixel(j->prm, j->gs, j->ws, j->hs, j->lut, j->gt, j->wt, j->ht, px, py, &c, &lv);
            if (j->coords) j->coords[i] = c;
            if (j->level) j->level[i] = lv;
            if (j->ct) {                                                   /* C_T[p] = C_S[s] */
                int64_t si = (int64_t)(c >> 16) * j->ws + (c & 0xFFFFu);
                memcpy(j->ct + 4 * i, j->cs + 4 * si, 4);
            }
        }
    }
    return NULL;
}

void or_stylize(const or_params* prm, const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                uint8_t* ct, uint32_t* coords, uint8_t* level, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    sty_job jobs[256];
    for (int32_t i = 0; i < nthreads; ++i) {
        sty_job j = {prm, cs, gs, ws, hs, lut, gt, wt, ht, ct, coords, level,
                     (int32_t)((int64_t)ht * i / nthreads), (int32_t)((int64_t)ht * (i + 1) / nthreads)};
        jobs[i] = j;
    }
    if (nthreads == 1) { sty_worker(&jobs[0]); return; }
    for (int32_t i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, sty_worker, &jobs[i]);
    for (int32_t i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------------------------ */
/* Voting (R13, R14).                                                  */
/* C_T[p] = average over target pixels q with |q - p|_inf <= r (clipped to the target)   */
/* of C_S[src(q) + (p - q)], skipping positions outside the source; per channel          */
/* floor((sum + floor(n/2)) / n).                                                        */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    const uint32_t* coords; int32_t wt, ht; const uint8_t* cs; int32_t ws, hs, r;
    uint8_t* ct; int32_t y_begin, y_end;
} vote_job;

static void* vote_worker(void* arg) {
    vote_job* j = (vote_job*)arg;
    for (int32_t py = j->y_begin; py < j->y_end; ++py) {
        for (int32_t px = 0; px < j->wt; ++px) {
            uint64_t sum[4] = {0, 0, 0, 0};
            uint64_t n = 0;
            for (int32_t qy = py - j->r; qy <= py + j->r; ++qy) {
                for (int32_t qx = px - j->r; qx <= px + j->r; ++qx) {
                    if (qx < 0 || qx >= j->wt || qy < 0 || qy >= j->ht) continue;
                    uint32_t src = j->coords[(int64_t)qy * j->wt + qx];
                    int32_t sx = (int32_t)(src & 0xFFFFu) + (px - qx);
                    int32_t sy = (int32_t)(src >> 16) + (py - qy);
                    if (sx < 0 || sx >= j->ws || sy < 0 || sy >= j->hs) continue;
                    const uint8_t* c = j->cs + 4 * ((int64_t)sy * j->ws + sx);
                    for (int32_t ch = 0; ch < 4; ++ch) sum[ch] += c[ch];
                    n += 1;
                }
            }
            uint8_t* out = j->ct + 4 * ((int64_t)py * j->wt + px);
            if (n == 0) { memset(out, 0, 4); continue; }   /* unreachable for valid coords */
            for (int32_t ch = 0; ch < 4; ++ch)
                out[ch] = (uint8_t)((sum[ch] + n / 2) / n);   /* n >= 1: q = p always counts */
        }
    }
    return NULL;
}

void or_vote(const uint32_t* coords, int32_t wt, int32_t ht, const uint8_t* cs, int32_t ws,
             int32_t hs, int32_t r, uint8_t* ct, int32_t nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    vote_job jobs[256];
    for (int32_t i = 0; i < nthreads; ++i) {
        vote_job j = {coords, wt, ht, cs, ws, hs, r, ct,
                      (int32_t)((int64_t)ht * i / nthreads), (int32_t)((int64_t)ht * (i + 1) / nthreads)};
        jobs[i] = j;
    }
    if (nthreads == 1) { vote_worker(&jobs[0]); return; }
    for (int32_t i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, vote_worker, &jobs[i]);
    for (int32_t i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------------------------ */
/* Alg. 1, the brute-force sequential synthesizer, as  */
/* a quality/statistics reference -- not a speed path.  Transcribed in the paper's order: */
/* target pixels p row-major; for an empty p, u* = the look-up of G_T[p] (line "u* =      */
/* argmin_u ||G_T[p] - G_S[u]||", the same look-up as Alg. 2, R11/R26); then every source */
/* pixel q row-major: if p + (q - u*) is inside the target (reading R27) and empty, and   */
/* e = ||G_T[p + (q - u*)] - G_S[q]|| < t, copy C_S[q] there.  Pixels left empty take the */
/* look-up fallback (level 0, as R12).  Filled pixels get level 1.                        */
/* ------------------------------------------------------------------------------------ */
void or_blit_bruteforce(const or_params* prm, const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                        const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                        uint8_t* ct, uint32_t* coords, uint8_t* level) {
    const int64_t npx = (int64_t)wt * ht;
    uint8_t* filled = (uint8_t*)calloc((size_t)npx, 1);
    for (int32_t py = 0; py < ht; ++py) {
        for (int32_t px = 0; px < wt; ++px) {
            if (filled[(int64_t)py * wt + px]) continue;                  /* "C_T[p] is empty" */
            const uint32_t u = lut_at(prm, lut, gs, ws, hs, gt + 4 * ((int64_t)py * wt + px));
            const int32_t ux = (int32_t)(u & 0xFFFFu), uy = (int32_t)(u >> 16);
            for (int32_t qy = 0; qy < hs; ++qy) {
                for (int32_t qx = 0; qx < ws; ++qx) {                     /* each q in C_S */
                    const int32_t tx = px + (qx - ux), ty = py + (qy - uy);
                    if (tx < 0 || tx >= wt || ty < 0 || ty >= ht) continue;  /* R27 */
                    const int64_t ti = (int64_t)ty * wt + tx;
                    if (filled[ti]) continue;
                    const uint8_t* gt_t = gt + 4 * ti;
                    const uint8_t* gs_q = gs + 4 * ((int64_t)qy * ws + qx);
                    if (prm->label_channel >= 0 && gt_t[prm->label_channel] != gs_q[prm->label_channel]) continue;
                    double e2 = 0.0;
                    for (int32_t c = 0; c < prm->C; ++c) {
                        if (c == prm->label_channel) continue;
                        double d = (double)gt_t[c] - (double)gs_q[c];
                        e2 += (double)prm->w[c] * d * d;
                    }
                    if (sqrt(e2) < prm->t) {                               /* e < t */
                        filled[ti] = 1;
                        coords[ti] = (uint32_t)qx | ((uint32_t)qy << 16);
                        if (level) level[ti] = 1;
                        if (ct) memcpy(ct + 4 * ti, cs + 4 * ((int64_t)qy * ws + qx), 4);
                    }
                }
            }
        }
    }
    for (int64_t i = 0; i < npx; ++i) {                                    /* never filled */
        if (filled[i]) continue;
        const uint32_t u = lut_at(prm, lut, gs, ws, hs, gt + 4 * i);
        coords[i] = u;
        if (level) level[i] = 0;
        if (ct) memcpy(ct + 4 * i, cs + 4 * ((int64_t)(u >> 16) * ws + (u & 0xFFFFu)), 4);
    }
    free(filled);
}
