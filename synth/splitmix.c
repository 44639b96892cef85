/* Counter-based splitmix64 input generator (C, host side) -- the same recipe
 * as synth/splitmix.py, for inputs too large for
 * numpy in test time.  Holds none of the method's arithmetic. */
#include <stdint.h>

static uint64_t mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t word(uint64_t stream, uint64_t i)
{
    uint64_t seed = (2209ull << 16) | stream;
    return mix(seed + (i + 1ull) * 0x9E3779B97F4A7C15ull);
}

void synth_raw(uint64_t stream, int64_t start, int64_t n, uint64_t *out)
{
    for (int64_t e = 0; e < n; ++e) out[e] = word(stream, (uint64_t)(start + e));
}

void synth_f32_unit(uint64_t stream, int64_t start, int64_t n, float *out)
{
    for (int64_t e = 0; e < n; ++e)
        out[e] = (float)((double)(word(stream, (uint64_t)(start + e)) >> 40) * 0x1.0p-24);
}

void synth_i64_sym(uint64_t stream, int64_t start, int64_t n, int64_t *out)
{
    for (int64_t e = 0; e < n; ++e)
        out[e] = (int64_t)(word(stream, (uint64_t)(start + e)) >> 35) - ((int64_t)1 << 28);
}
