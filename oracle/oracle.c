/*
 * oracle/oracle.c -- plain, slow, obviously correct CPU oracle for the stable
 * merge and the stable merge sort of arXiv 1202.6575.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1202_6575_b200/csrc) and includes nothing from it.
 *
 * The method reaches exactly the plain stable merge (§2, Theorem
 * L366-371 with the correctness argument L343-357), so the oracle is that
 * definition written out, not the parallel algorithm:
 *
 *   oracle_merge_*   two pointers; emit A[i] when A[i] <= B[j], else B[j]
 *                    ("all (repeated) elements a from A are ordered before
 *                    elements a from B").
 *   oracle_sort_*    bottom-up stable merge sort: runs of width 1, 2, 4, ...
 *                    merged pairwise with the left run playing A (§3
 *                    L403-416: the unique stable sort).
 *   oracle_rank_low_*  / oracle_rank_high_*   rank_low(x,X) = unique i with
 *                    X[i-1] < x <= X[i]; rank_high(x,X) = unique j with
 *                    X[j-1] <= x < X[j]  (sentinels
 *                    X[-1]=-inf, X[len]=+inf, L69-71), by plain binary search.
 *   oracle_positions_*  the closed form of PAPER.md L158-166: A[i] goes to
 *                    C[i + rank_low(A[i],B)], B[j] to C[j + rank_high(B[j],A)].
 *
 * Keys: u32 / i32 / i64 / u64 with the natural (unsigned or signed) order;
 * f32 / f64 with IEEE 754 totalOrder; u128 unsigned
 * 128-bit (= (high, low) 64-bit tuples, lexicographic); the desc_*
 * functions use the reversed order (descending keys, still ties to A).
 * Payloads: uint32, travelling with their key; NULL payload pointers mean
 * keys only.  *_wide_*: payloads of any w bytes (structs), same definition.  Sizes are int64.  No error paths: callers pass valid sizes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* The key order "<=": natural for integer keys; IEEE 754
 * totalOrder for floating-point keys, through an integer key: the bit
 * pattern read as a signed integer, with the magnitude bits of negative
 * values inverted (so -NaN < -inf < ... < -0.0 < +0.0 < ... < +inf < +NaN). */
static int32_t tot_f32(float x) { int32_t i; memcpy(&i, &x, 4); return i < 0 ? i ^ 0x7fffffff : i; }
static int64_t tot_f64(double x) { int64_t i; memcpy(&i, &x, 8); return i < 0 ? i ^ 0x7fffffffffffffffLL : i; }
#define LE_INT(a, b) ((a) <= (b))
#define LT_INT(a, b) ((a) < (b))
#define LE_F32(a, b) (tot_f32(a) <= tot_f32(b))
#define LT_F32(a, b) (tot_f32(a) < tot_f32(b))
#define LE_F64(a, b) (tot_f64(a) <= tot_f64(b))
#define LT_F64(a, b) (tot_f64(a) < tot_f64(b))

#define DEFINE_ORACLE(SUF, K, LE, LT)                                                 \
                                                                                      \
/* Stable two-way merge, ties to A.  vc may be NULL (keys only). */                  \
void oracle_merge_##SUF(const K *a, const uint32_t *va, int64_t n,                   \
                        const K *b, const uint32_t *vb, int64_t m,                   \
                        K *c, uint32_t *vc)                                          \
{                                                                                     \
    int64_t i = 0, j = 0, k = 0;                                                     \
    while (i < n && j < m) {                                                         \
        if (LE(a[i], b[j])) {             /* tie -> A first */                       \
            c[k] = a[i];                                                             \
            if (vc) vc[k] = va[i];                                                   \
            i++;                                                                     \
        } else {                                                                     \
            c[k] = b[j];                                                             \
            if (vc) vc[k] = vb[j];                                                   \
            j++;                                                                     \
        }                                                                            \
        k++;                                                                         \
    }                                                                                \
    while (i < n) { c[k] = a[i]; if (vc) vc[k] = va[i]; i++; k++; }                 \
    while (j < m) { c[k] = b[j]; if (vc) vc[k] = vb[j]; j++; k++; }                 \
}                                                                                     \
                                                                                      \
/* Bottom-up stable merge sort in place (result in keys/vals). */                   \
int oracle_sort_##SUF(K *keys, uint32_t *vals, int64_t N)                            \
{                                                                                     \
    K *src = keys, *dst;                                                             \
    uint32_t *vsrc = vals, *vdst = NULL;                                             \
    int64_t width;                                                                   \
    if (N <= 1) return 0;                                                            \
    dst = (K *)malloc((size_t)N * sizeof(K));                                        \
    if (!dst) return -1;                                                             \
    if (vals) {                                                                      \
        vdst = (uint32_t *)malloc((size_t)N * sizeof(uint32_t));                     \
        if (!vdst) { free(dst); return -1; }                                         \
    }                                                                                \
    K *kbuf = dst; uint32_t *vbuf = vdst;                                            \
    for (width = 1; width < N; width *= 2) {                                         \
        int64_t lo;                                                                  \
        for (lo = 0; lo < N; lo += 2 * width) {                                      \
            int64_t mid = lo + width < N ? lo + width : N;                           \
            int64_t hi = lo + 2 * width < N ? lo + 2 * width : N;                    \
            /* left run [lo,mid) plays A, right run [mid,hi) plays B */             \
            oracle_merge_##SUF(src + lo, vsrc ? vsrc + lo : NULL, mid - lo,          \
                               src + mid, vsrc ? vsrc + mid : NULL, hi - mid,        \
                               dst + lo, vsrc ? vdst + lo : NULL);                   \
        }                                                                            \
        { K *t = src; src = dst; dst = t; }                                          \
        { uint32_t *t = vsrc; vsrc = vdst; vdst = t; }                               \
    }                                                                                \
    if (src != keys) {                                                               \
        memcpy(keys, src, (size_t)N * sizeof(K));                                    \
        if (vals) memcpy(vals, vsrc, (size_t)N * sizeof(uint32_t));                  \
    }                                                                                \
    free(kbuf);                                                                      \
    free(vbuf);                                                                      \
    return 0;                                                                        \
}                                                                                     \
                                                                                      \
/* rank_low(x, X): number of elements of X strictly less than x. */                 \
int64_t oracle_rank_low_##SUF(K x, const K *X, int64_t len)                          \
{                                                                                     \
    int64_t lo = 0, hi = len;       /* answer in [lo, hi] */                        \
    while (lo < hi) {                                                                \
        int64_t mid = lo + (hi - lo) / 2;                                            \
        if (LT(X[mid], x)) lo = mid + 1; else hi = mid;                              \
    }                                                                                \
    return lo;                                                                       \
}                                                                                     \
                                                                                      \
/* rank_high(x, X): number of elements of X less than or equal to x. */             \
int64_t oracle_rank_high_##SUF(K x, const K *X, int64_t len)                         \
{                                                                                     \
    int64_t lo = 0, hi = len;                                                        \
    while (lo < hi) {                                                                \
        int64_t mid = lo + (hi - lo) / 2;                                            \
        if (LE(X[mid], x)) lo = mid + 1; else hi = mid;                              \
    }                                                                                \
    return lo;                                                                       \
}                                                                                     \
                                                                                      \
/* Closed-form output positions. */                             \
void oracle_positions_##SUF(const K *a, int64_t n, const K *b, int64_t m,            \
                            int64_t *pos_a, int64_t *pos_b)                          \
{                                                                                     \
    int64_t i, j;                                                                    \
    for (i = 0; i < n; i++) pos_a[i] = i + oracle_rank_low_##SUF(a[i], b, m);        \
    for (j = 0; j < m; j++) pos_b[j] = j + oracle_rank_high_##SUF(b[j], a, n);       \
}                                                                                     \
                                                                                      \
/* Stable merge with payloads of w bytes each (wide   \
 * and struct payloads): the same two-pointer definition, the w payload       \
 * bytes travelling with their key. */                                        \
void oracle_merge_wide_##SUF(const K *a, const void *va, int64_t n,              \
                             const K *b, const void *vb, int64_t m,              \
                             K *c, void *vc, int64_t w)                          \
{                                                                                     \
    int64_t i = 0, j = 0, k = 0;                                                     \
    const char *pa = (const char *)va, *pb = (const char *)vb;                       \
    char *pc = (char *)vc;                                                           \
    while (i < n || j < m) {                                                         \
        if (j >= m || (i < n && LE(a[i], b[j]))) {    /* tie -> A first */           \
            c[k] = a[i];                                                             \
            memcpy(pc + k * w, pa + i * w, (size_t)w);                               \
            i++;                                                                     \
        } else {                                                                     \
            c[k] = b[j];                                                             \
            memcpy(pc + k * w, pb + j * w, (size_t)w);                               \
            j++;                                                                     \
        }                                                                            \
        k++;                                                                         \
    }                                                                                \
}                                                                                     \
                                                                                      \
/* Bottom-up stable merge sort in place with w-byte payloads. */                    \
int oracle_sort_wide_##SUF(K *keys, void *vals, int64_t N, int64_t w)              \
{                                                                                     \
    K *src = keys, *dst;                                                             \
    char *vsrc = (char *)vals, *vdst;                                                \
    int64_t width;                                                                   \
    if (N <= 1) return 0;                                                            \
    dst = (K *)malloc((size_t)N * sizeof(K));                                        \
    vdst = (char *)malloc((size_t)(N * w));                                          \
    if (!dst || !vdst) { free(dst); free(vdst); return -1; }                         \
    K *kbuf = dst; char *vbuf = vdst;                                                \
    for (width = 1; width < N; width *= 2) {                                         \
        int64_t lo;                                                                  \
        for (lo = 0; lo < N; lo += 2 * width) {                                      \
            int64_t mid = lo + width < N ? lo + width : N;                           \
            int64_t hi = lo + 2 * width < N ? lo + 2 * width : N;                    \
            oracle_merge_wide_##SUF(src + lo, vsrc + lo * w, mid - lo,               \
                                    src + mid, vsrc + mid * w, hi - mid,             \
                                    dst + lo, vdst + lo * w, w);                     \
        }                                                                            \
        { K *t = src; src = dst; dst = t; }                                          \
        { char *t = vsrc; vsrc = vdst; vdst = t; }                                   \
    }                                                                                \
    if (src != keys) {                                                               \
        memcpy(keys, src, (size_t)N * sizeof(K));                                    \
        memcpy(vals, vsrc, (size_t)(N * w));                                         \
    }                                                                                \
    free(kbuf);                                                                      \
    free(vbuf);                                                                      \
    return 0;                                                                        \
}                                                                                     \
                                                                                      \
/* Positions for a sample of indices only (full-size parity checks). */             \
void oracle_positions_sample_##SUF(const K *a, int64_t n, const K *b, int64_t m,     \
                                   const int64_t *ia, int64_t na, int64_t *pos_a,    \
                                   const int64_t *jb, int64_t nb, int64_t *pos_b)    \
{                                                                                     \
    int64_t t;                                                                       \
    for (t = 0; t < na; t++) pos_a[t] = ia[t] + oracle_rank_low_##SUF(a[ia[t]], b, m);\
    for (t = 0; t < nb; t++) pos_b[t] = jb[t] + oracle_rank_high_##SUF(b[jb[t]], a, n);\
}

/* Descending order: the paper's method for an
 * arbitrary total order "<=", instantiated with the reversed
 * order a <=' b  <=>  b <= a.  Everything above is unchanged: stability is
 * still "A before B on ties" (L160-163) under the reversed order. */
#define LE_REV(LE, a, b) LE(b, a)
#define LE_D_INT(a, b) LE_REV(LE_INT, a, b)
#define LT_D_INT(a, b) LE_REV(LT_INT, a, b)
#define LE_D_F32(a, b) LE_REV(LE_F32, a, b)
#define LT_D_F32(a, b) LE_REV(LT_F32, a, b)
#define LE_D_F64(a, b) LE_REV(LE_F64, a, b)
#define LT_D_F64(a, b) LE_REV(LT_F64, a, b)

DEFINE_ORACLE(u32, uint32_t, LE_INT, LT_INT)
DEFINE_ORACLE(i32, int32_t, LE_INT, LT_INT)
DEFINE_ORACLE(i64, int64_t, LE_INT, LT_INT)
DEFINE_ORACLE(u64, uint64_t, LE_INT, LT_INT)
DEFINE_ORACLE(f32, float, LE_F32, LT_F32)
DEFINE_ORACLE(f64, double, LE_F64, LT_F64)
/* 128-bit keys (128-bit keys and (key, tie) tuples):
 * unsigned, i.e. the lexicographic order of (high 64 bits, low 64 bits). */
typedef unsigned __int128 u128_t;
DEFINE_ORACLE(u128, u128_t, LE_INT, LT_INT)
DEFINE_ORACLE(desc_u128, u128_t, LE_D_INT, LT_D_INT)
/* the rank functions with the key passed by pointer (no 128-bit scalars in ctypes) */
int64_t oracle_rank_low_ptr_u128(const u128_t *x, const u128_t *X, int64_t len) { return oracle_rank_low_u128(*x, X, len); }
int64_t oracle_rank_high_ptr_u128(const u128_t *x, const u128_t *X, int64_t len) { return oracle_rank_high_u128(*x, X, len); }
int64_t oracle_rank_low_ptr_desc_u128(const u128_t *x, const u128_t *X, int64_t len) { return oracle_rank_low_desc_u128(*x, X, len); }
int64_t oracle_rank_high_ptr_desc_u128(const u128_t *x, const u128_t *X, int64_t len) { return oracle_rank_high_desc_u128(*x, X, len); }

DEFINE_ORACLE(desc_u32, uint32_t, LE_D_INT, LT_D_INT)
DEFINE_ORACLE(desc_i32, int32_t, LE_D_INT, LT_D_INT)
DEFINE_ORACLE(desc_i64, int64_t, LE_D_INT, LT_D_INT)
DEFINE_ORACLE(desc_u64, uint64_t, LE_D_INT, LT_D_INT)
DEFINE_ORACLE(desc_f32, float, LE_D_F32, LT_D_F32)
DEFINE_ORACLE(desc_f64, double, LE_D_F64, LT_D_F64)
