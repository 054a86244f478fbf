/* examples/decode_host.c -- the C ABI without Python or PyTorch: decode a small batch of BSID frames
 * (q = 8, n = 7, N = 10: BASELINE config C1's code shape) from HOST buffers with
 * bsidmap_decode_batch_host and report the symbol error rate of the hard decisions.
 *
 *   make examples/decode_host && LD_LIBRARY_PATH=paper_1802_08483_b200 ./examples/decode_host
 *
 * The channel is the literal event loop of P:90-100 (insertion of a random bit w.p. Pi, deletion
 * w.p. Pd, transmission w.p. 1 - Pi - Pd with substitution w.p. Ps), driven by a small LCG. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "bsidmap.h"

static uint64_t s_state = 0x1802084830ull;
static double urand(void) { /* 53-bit uniform in [0, 1) */
  s_state = s_state * 6364136223846793005ull + 1442695040888963407ull;
  return (double)(s_state >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
  enum { q = 8, n = 7, N = 10, F = 256, WPF = 4 };
  const double Pi = 0.01, Pd = 0.01, Ps = 0.0;
  int mn_lo, mn_hi, mt_lo, mt_hi;
  if (bsidmap_state_space(n, N, Pi, Pd, 1e-10, &mn_lo, &mn_hi, &mt_lo, &mt_hi) != BSIDMAP_OK) return 1;
  /* time-varying random injective codebook C_i(D) */
  uint32_t C[N * q];
  for (int i = 0; i < N; i++)
    for (int D = 0; D < q; D++) {
      uint32_t w;
      int dup;
      do {
        w = (uint32_t)(urand() * (1u << n));
        dup = 0;
        for (int e = 0; e < D; e++) dup |= C[i * q + e] == w;
      } while (dup);
      C[i * q + D] = w;
    }
  bsidmap_decoder *d = NULL;
  if (bsidmap_create(&d, q, n, N, C, Pi, Pd, Ps, mn_lo, mn_hi, mt_lo, mt_hi, BSIDMAP_MODE_AUTO, 0) != BSIDMAP_OK) {
    fprintf(stderr, "create: %s\n", bsidmap_last_error(NULL));
    return 1;
  }
  uint32_t *rx = calloc((size_t)F * WPF, sizeof(uint32_t));
  int64_t *off = malloc(sizeof(int64_t) * F);
  int32_t *rho = malloc(sizeof(int32_t) * F), *st = malloc(sizeof(int32_t) * F), *msg = malloc(sizeof(int32_t) * F * N);
  float *L = malloc(sizeof(float) * F * N * q);
  for (int f = 0; f < F; f++) {
    int len;
    do { /* redraw frames whose end drift leaves [m_tau^-, m_tau^+] (reading R13) */
      memset(rx + (size_t)f * WPF, 0, WPF * 4);
      len = 0;
      for (int i = 0; i < N; i++) {
        const int D = (int)(urand() * q);
        msg[f * N + i] = D;
        for (int t = 0; t < n; t++) {
          const uint32_t x = (C[i * q + D] >> t) & 1u;
          for (;;) {
            const double u = urand();
            if (u < Pi) { /* insertion of a random bit, then the same bit is tried again */
              if (urand() < 0.5 && len < WPF * 32) rx[(size_t)f * WPF + len / 32] |= 1u << (len % 32);
              len++;
              continue;
            }
            if (u < Pi + Pd) break; /* deletion */
            const uint32_t y = (urand() < Ps) ? x ^ 1u : x;
            if (y && len < WPF * 32) rx[(size_t)f * WPF + len / 32] |= 1u << (len % 32);
            len++;
            break;
          }
        }
      }
    } while (len - n * N < mt_lo || len - n * N > mt_hi || len > WPF * 32);
    rho[f] = len;
    off[f] = (int64_t)f * WPF;
  }
  if (bsidmap_decode_batch_host(d, F, rx, (size_t)F * WPF, off, rho, NULL, L, st, NULL) != BSIDMAP_OK) {
    fprintf(stderr, "decode: %s\n", bsidmap_last_error(d));
    return 1;
  }
  long errors = 0, ok = 0;
  for (int f = 0; f < F; f++) {
    ok += st[f] == BSIDMAP_FRAME_OK;
    for (int i = 0; i < N; i++) {
      const float *row = L + ((size_t)f * N + i) * q;
      int best = 0;
      for (int D = 1; D < q; D++)
        if (row[D] > row[best]) best = D;
      errors += best != msg[f * N + i];
    }
  }
  printf("decoded %d frames (%ld ok), symbol error rate %.5f, launches %ld\n", F, ok, (double)errors / (F * N),
         bsidmap_last_launch_count(d));
  bsidmap_destroy(d);
  free(rx); free(off); free(rho); free(st); free(msg); free(L);
  return ok == F ? 0 : 2;
}
