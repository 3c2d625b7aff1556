// Host-side use of the CUDA toolkit's own Philox4x32-10 (curand_philox4x32_x.h
// has an NV_IS_HOST path).  Library cross-check for the oracle's Philox —
// tests/test_oracle_pins.py compiles this with g++ and compares outputs.
#define QUALIFIERS static inline
#include <cstdio>
#include <cstdlib>
#include <vector_types.h>
#include <curand_philox4x32_x.h>
int main(int argc, char** argv) {
    // reads lines "c0 c1 c2 c3 k0 k1" (hex) from stdin, prints the 4 outputs
    unsigned c0, c1, c2, c3, k0, k1;
    while (scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
        uint4 c = {c0, c1, c2, c3};
        uint2 k = {k0, k1};
        uint4 r = curand_Philox4x32_10(c, k);
        printf("%08x %08x %08x %08x\n", r.x, r.y, r.z, r.w);
    }
    return 0;
}
