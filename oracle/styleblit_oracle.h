/*
 * styleblit_oracle.h -- CPU ORACLE for StyleBlit (arXiv 1807.03249), TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain, slow, single-threaded-by-default transcription of the paper's
 * Algorithm 2 ("ParallelStyleBlit", sec. 3.2) and of the voting
 * step.  It exists to prove the CUDA path correct.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  It shares no code, header, table or constant generator with
 * paper_1807_03249_b200/ (the product), and the product never loads it.
 *
 * Every open point of the paper is fixed by a numbered reading listed in
 * DESIGN.md ("Readings"); the numbers R1..R27 below refer to that list.
 *
 * Images: row-major, 4 bytes per pixel (uint8 x4), pixel (x,y) at byte 4*(y*W+x).
 * Coordinates returned packed as x | y<<16 (uint32).
 */
#ifndef STYLEBLIT_ORACLE_H
#define STYLEBLIT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Oracle parameters (the paper's inputs t and L, plus readings). */
typedef struct {
    double   t;               /* threshold t in 8-bit guide units (R2); accept iff e < t (R3) */
    int32_t  L;               /* number of levels, level l uses spacing h = 2^l (R4)           */
    int32_t  C;               /* guide channels used by the error e (R11, R18): 2..4           */
    uint32_t seed;            /* jitter-table seed (R5, R19)                                   */
    int32_t  zero_jitter;     /* 1: RandomJitterTable == 0 everywhere (test hook)              */
    int32_t  w[4];            /* per-channel weights of e^2 (SPEC compose_guides)   */
    int32_t  label_channel;   /* -1: none; else a segmentation label byte   */
    int32_t  lut_rgb;         /* 1: u* by exact search over channels 0..2 (R26), lut unused    */
} or_params;

/* R5 / SURVEY App. A: the stateless hash that realises RandomJitterTable. */
uint32_t or_lowbias32(uint32_t x);
uint32_t or_cell_hash(int32_t bx, int32_t by, int32_t l, uint32_t seed);
/* j = RandomJitterTable[b] at level l, as the two real numbers in [0,1) (16-bit quantised). */
void or_jitter(int32_t bx, int32_t by, int32_t l, uint32_t seed, int32_t zero_jitter,
               double* jx, double* jy);

/* Alg. 2 SeedPoint(p, h) with an explicit jitter; used for the
 * SPEC forced-jitter example.  b = floor(p/h) (floor toward -inf). */
void or_seed_point_j(int32_t px, int32_t py, int32_t h, double jx, double jy,
                     int32_t* sx, int32_t* sy);
/* Alg. 2 SeedPoint(p, 2^l) with the table of R5. */
void or_seed_point(int32_t px, int32_t py, int32_t l, uint32_t seed, int32_t zero_jitter,
                   int32_t* sx, int32_t* sy);
/* Alg. 2 NearestSeed(p, 2^l): raw (unclamped) seed. */
void or_nearest_seed(int32_t px, int32_t py, int32_t l, uint32_t seed, int32_t zero_jitter,
                     int32_t* qx, int32_t* qy);

/* Guide look-up: u* = argmin_u ||g - G_S[u]|| over channels 0,1
 * (R10, R11); ties -> smallest row-major source index.  Returns x | y<<16. */
uint32_t or_lut_entry(const uint8_t* gs, int32_t ws, int32_t hs, int32_t g0, int32_t g1);
/* The full 256x256 table, LUT[g0 | g1<<8].  nthreads>1 splits the KEYS over threads;
 * every entry is still computed by or_lut_entry. */
void or_build_lut(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut, int32_t nthreads);

/* Exact three-channel guide search ("or a tree search", reading R26):
 * u* = argmin_u over channels 0,1,2, ties -> smallest row-major index.  x | y<<16. */
uint32_t or_lut3_entry(const uint8_t* gs, int32_t ws, int32_t hs, int32_t g0, int32_t g1, int32_t g2);
/* or_lut3_entry for n keys g0 | g1<<8 | g2<<16 (nthreads split the list). */
void or_lut3_entries(const uint8_t* gs, int32_t ws, int32_t hs, const uint32_t* keys, int64_t n,
                     uint32_t* out, int32_t nthreads);

/* Alg. 2 ParallelStyleBlit for one target pixel with the fallback of
 * R12.  Writes the source coordinate (x | y<<16) and the accepting level (0 = fallback). */
void or_stylize_pixel(const or_params* prm, const uint8_t* gs, int32_t ws, int32_t hs,
                      const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                      int32_t px, int32_t py, uint32_t* coord, uint8_t* level);
/* Every target pixel, rows [0,ht) (nthreads>1 splits rows; per-pixel function unchanged).
 * ct (may be NULL) receives the blit C_T[p] = C_S[coords[p]]. */
void or_stylize(const or_params* prm, const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                uint8_t* ct, uint32_t* coords, uint8_t* level, int32_t nthreads);

/* Voting (R13, R14): average of co-located pixels of the patches of
 * radius r that overlap p.  r = 0 is the blit. */
void or_vote(const uint32_t* coords, int32_t wt, int32_t ht, const uint8_t* cs, int32_t ws,
             int32_t hs, int32_t r, uint8_t* ct, int32_t nthreads);

/* Alg. 1, the brute-force sequential synthesizer, a statistics reference
 * (SURVEY 8(f) #4).  coords/ct/level as or_stylize; level 1 = copied, 0 = look-up fallback. */
void or_blit_bruteforce(const or_params* prm, const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                        const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht,
                        uint8_t* ct, uint32_t* coords, uint8_t* level);

const char* or_version(void);

#ifdef __cplusplus
}
#endif
#endif
