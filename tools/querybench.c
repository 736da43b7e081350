/* querybench.c — native Bloom-bank query latency (the paper's 0.4 us/lookup).
 *   gcc -O2 -o /tmp/querybench tools/querybench.c -Lpaper_2408_11417_b200 -lskpp \
 *       -Wl,-rpath,$PWD/paper_2408_11417_b200 && /tmp/querybench
 * Seven filters of the reference default geometry (capacity 10000, fp 0.01: 95,872 bits,
 * k = 7), half the bits set, seeds by bank position; times skpp_bank_snapshot_query on a
 * stream of distinct (m, n, k) keys, one thread. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

uint64_t skpp_bank_snapshot_query(const void* snap, uint64_t m, uint64_t n, uint64_t k);
void* skpp_bank_snapshot(const uint8_t* bits, const uint32_t* seeds, uint32_t n_filters, uint64_t m_bits,
                         uint32_t k_hashes);
void skpp_bank_snapshot_free(void* snap);

int main(void) {
  const uint32_t P = 7, K = 7;
  const uint64_t m_bits = 95872;
  uint8_t* bits = malloc(P * m_bits / 8);
  uint32_t seeds[7];
  for (uint32_t i = 0; i < P; ++i) seeds[i] = (uint32_t)(0x9E3779B9ull * (i + 1));
  srand(1);
  for (uint64_t i = 0; i < P * m_bits / 8; ++i) bits[i] = (uint8_t)rand();
  void* snap = skpp_bank_snapshot(bits, seeds, P, m_bits, K);
  if (!snap) { printf("snapshot failed\n"); return 1; }
  const uint64_t N = 20000000;
  uint64_t acc = 0;
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (uint64_t i = 0; i < N; ++i) acc += skpp_bank_snapshot_query(snap, 1 + (i & 8191), 64 + (i >> 13), 4096);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  double ns = ((t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec)) / (double)N;
  printf("skpp_bank_snapshot_query: %.1f ns per query (7 filters, k=7, 1 thread; checksum %llu)\n", ns,
         (unsigned long long)acc);
  skpp_bank_snapshot_free(snap);
  free(bits);
  return 0;
}
