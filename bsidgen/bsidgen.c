/*
 * bsidgen.c -- seeded synthetic inputs for the BSID MAP decoder (shared by
 * the oracle tests, the CUDA parity tests and bench.py).
 *
 * This module holds NONE of the decoder's arithmetic: it draws codebooks,
 * messages, channel outputs and priors.  Every random number comes from a
 * counter-based stream keyed by (seed, stream id, index), so a frame's
 * content depends only on (seed, global frame index) -- identical whatever
 * the number of GPUs or threads.
 *
 *   codebook : per position i, q distinct n-bit words uniform without
 *              replacement (random injective C_i); bit t (LSB = 0)
 *              is the t-th transmitted bit (reading R15)
 *   message  : D_i ~ U[0, q)
 *   channel  : the literal per-time-step BSID event loop:
 *              insertion Pi (uniform random bit, stay at t), deletion Pd,
 *              transmission Pt = 1 - Pi - Pd with substitution Ps.
 *              Frames whose end drift rho - tau falls outside
 *              [mt_lo, mt_hi] are redrawn and counted.
 *   priors   : "as in iterative decoding": P(D_i = D) proportional
 *              to exp(2 [D = D_i] + g), g ~ N(0,1)  (documented choice)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct {
    uint64_t key, ctr;
} rng_t;

static inline rng_t rng_make(uint64_t seed, uint64_t stream, uint64_t index)
{
    rng_t r;
    r.key = splitmix64(splitmix64(seed ^ 0x1802084830000000ull) ^ splitmix64(stream * 0x632BE59BD9B4E019ull + 1))
            ^ splitmix64(index + 0x2545F4914F6CDD1Dull);
    r.ctr = 0;
    return r;
}

static inline uint64_t rng_next(rng_t *r)
{
    return splitmix64(r->key + 0x9E3779B97F4A7C15ull * (++r->ctr));
}

/* uniform double in [0, 1) with 53 random bits */
static inline double rng_unif(rng_t *r)
{
    return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}

static inline uint64_t rng_below(rng_t *r, uint64_t bound)
{
    /* rejection sampling for an unbiased draw in [0, bound) */
    uint64_t lim = UINT64_MAX - (UINT64_MAX % bound);
    uint64_t v;
    do {
        v = rng_next(r);
    } while (v >= lim);
    return v % bound;
}

enum { STREAM_CODEBOOK = 1, STREAM_MESSAGE = 2, STREAM_CHANNEL = 3, STREAM_PRIORS = 4 };

/* q distinct words per position (uniform without replacement). Returns 0 or -1. */
int gen_codebook(uint64_t seed, int N, int q, int n, uint32_t *C)
{
    int i, D, E;
    uint64_t space;
    if (n < 1 || n > 32 || q < 1 || N < 1)
        return -1;
    space = (uint64_t)1 << n;
    if ((uint64_t)q > space)
        return -1;
    for (i = 0; i < N; i++) {
        rng_t r = rng_make(seed, STREAM_CODEBOOK, (uint64_t)i);
        uint32_t *row = C + (size_t)i * q;
        for (D = 0; D < q; D++) {
            uint32_t w;
            int dup;
            do {
                w = (uint32_t)rng_below(&r, space);
                dup = 0;
                for (E = 0; E < D; E++)
                    if (row[E] == w) {
                        dup = 1;
                        break;
                    }
            } while (dup);
            row[D] = w;
        }
    }
    return 0;
}

/*
 * Frames [first, first + count): message D[f][N], packed received words
 * rx[f][words_per_frame] (LSB-first, zero padded), rho[f].  Bits beyond
 * words_per_frame * 32 are impossible because mt_hi bounds rho - tau.
 * Returns the total number of channel redraws, or -1 on bad arguments.
 */
int64_t gen_frames(uint64_t seed, int64_t first, int count, int N, int q, int n,
                   const uint32_t *C, double Pi, double Pd, double Ps,
                   int mt_lo, int mt_hi, int words_per_frame,
                   int32_t *msg, uint32_t *rx, int32_t *rho)
{
    const int tau = n * N;
    int64_t redraws = 0;
    int f, i, t;
    if ((int64_t)words_per_frame * 32 < (int64_t)tau + mt_hi || !(Pi + Pd < 1.0))
        return -1;
    for (f = 0; f < count; f++) {
        const int64_t gf = first + f;
        rng_t rm = rng_make(seed, STREAM_MESSAGE, (uint64_t)gf);
        rng_t rc = rng_make(seed, STREAM_CHANNEL, (uint64_t)gf);
        int32_t *m = msg + (size_t)f * N;
        uint32_t *w = rx + (size_t)f * words_per_frame;
        for (i = 0; i < N; i++)
            m[i] = (int32_t)rng_below(&rm, (uint64_t)q);
        for (;;) {
            int64_t out = 0;
            memset(w, 0, sizeof(uint32_t) * (size_t)words_per_frame);
            for (i = 0; i < N; i++) {
                const uint32_t word = C[(size_t)i * q + m[i]];
                for (t = 0; t < n; t++) {
                    const uint32_t xb = (word >> t) & 1u;
                    for (;;) { /* events at time t */
                        double u = rng_unif(&rc);
                        uint32_t ob;
                        if (u < Pi) { /* insertion: random bit, stay at t */
                            ob = (uint32_t)(rng_next(&rc) >> 63);
                        } else if (u < Pi + Pd) { /* deletion: advance */
                            break;
                        } else { /* transmission (+ substitution Ps): advance */
                            ob = xb ^ (uint32_t)(rng_unif(&rc) < Ps);
                        }
                        if (out < (int64_t)words_per_frame * 32)
                            w[out >> 5] |= ob << (out & 31);
                        out++;
                        if (u >= Pi)
                            break;
                    }
                }
            }
            if (out - tau >= mt_lo && out - tau <= mt_hi) {
                rho[f] = (int32_t)out;
                break;
            }
            redraws++;
        }
    }
    return redraws;
}

/* Non-uniform priors [count][N][q] (rows sum to 1), see header. */
int gen_priors(uint64_t seed, int64_t first, int count, int N, int q, const int32_t *msg, float *pri)
{
    int f, i, D;
    for (f = 0; f < count; f++) {
        rng_t r = rng_make(seed, STREAM_PRIORS, (uint64_t)(first + f));
        for (i = 0; i < N; i++) {
            double v[4096], s = 0.0;
            if (q > 4096)
                return -1;
            for (D = 0; D < q; D++) {
                /* Box-Muller standard normal */
                double u1 = rng_unif(&r), u2 = rng_unif(&r);
                double g = sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
                v[D] = exp(2.0 * (D == msg[(size_t)f * N + i]) + g);
                s += v[D];
            }
            for (D = 0; D < q; D++)
                pri[((size_t)f * N + i) * q + D] = (float)(v[D] / s);
        }
    }
    return 0;
}
