// Host harness (test infrastructure): the reference-order closed form of
// gs_refsum.cuh, compiled for the host, evaluated on (s0, a, c) triples read
// from stdin; prints the result bits.  tests/test_refsum_closed_form.py
// compares them with np.add.accumulate (the reference's np.bincount order).
#include <cstdio>
#include <cinttypes>
#include "../../paper_2104_00303_b200/csrc/gs_refsum.cuh"

int main() {
  unsigned long long sb, ab, c;
  while (scanf("%llx %llx %llu", &sb, &ab, &c) == 3) {
    double s, a;
    memcpy(&s, &sb, 8);
    memcpy(&a, &ab, 8);
    const double r = gs::seqsum_mag_from(s, a, c);
    unsigned long long rb;
    memcpy(&rb, &r, 8);
    printf("%016llx\n", rb);
  }
  return 0;
}
