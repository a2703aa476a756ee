/*
 * synth_gen.c — the counter-based input generator of synth.py (splitmix64 of the element index
 * under a key) written in plain C with OpenMP, for drawing the multi-GB full-batch inputs on the
 * host quickly.  Seeded input generation only: none of the method's arithmetic lives here.  It is
 * checked against synth.counter_codes (the torch implementation) by tests/test_synth.py.
 */
#include <stdint.h>

static inline uint64_t sg_hash(uint64_t idx, uint64_t key)
{
    uint64_t z = idx * 0x9E3779B97F4A7C15ull + key;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* out[i] = code of element start + i: dist 0 uniform U{0..3} (low 2 bits), dist 1 ReLU-skewed
 * (P(0) = 1/2 from the low 32 bits r < 2^31, else 1 + floor((r - 2^31) * 3 / 2^31)). */
void sg_counter_codes(int64_t start, int64_t count, uint64_t key, int32_t dist, uint8_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const uint32_t r = (uint32_t)sg_hash((uint64_t)(start + i), key);
        uint8_t c;
        if (dist == 0)
            c = (uint8_t)(r & 3u);
        else
            c = r < 0x80000000u ? 0 : (uint8_t)(1u + (uint32_t)(((uint64_t)(r - 0x80000000u) * 3u) >> 31));
        out[i] = c;
    }
}
