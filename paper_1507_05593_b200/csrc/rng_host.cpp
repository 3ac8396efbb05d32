// Host side of the device Gaussian sketch generator: the seeding chain the
// reference uses for every sketch (factor.py:324-326 `_block_seed`, then
// kernels.py:85-92 `np.random.Generator(np.random.PCG64(seed))`), restated in C++:
//
//   seed  = SeedSequence((master,) + tags).generate_state(1, uint64)[0]
//   PCG64(seed): SeedSequence(seed).generate_state(4, uint64) -> (initstate, initseq)
//                inc = initseq << 1 | 1; state = 0; step; state += initstate; step
//
// SeedSequence is O'Neill's seed_seq_fe hash (numpy/random/bit_generator.pyx,
// pool size 4); PCG64 is the 128-bit LCG with the XSL-RR output.  Both are
// integer-exact; tests/test_rng.py compares every word with numpy.
#include <cstdint>
#include <vector>

#include "../../include/rsc_b200.h"

namespace {

typedef unsigned __int128 u128;

constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
constexpr uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16;
constexpr int POOL = 4;

const u128 PCG_MULT = ((u128)0x2360ed051fc65da4ULL << 64) | 0x4385df649fccf645ULL;

inline uint32_t hashmix(uint32_t v, uint32_t &hc) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    v ^= v >> XSHIFT;
    return v;
}

inline uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> XSHIFT;
    return r;
}

// numpy's _int_to_uint32_array: little-endian 32-bit words, 0 -> [0]
void push_int(std::vector<uint32_t> &e, uint64_t v) {
    if (v == 0) {
        e.push_back(0);
        return;
    }
    while (v) {
        e.push_back((uint32_t)v);
        v >>= 32;
    }
}

void seed_seq_words(const std::vector<uint32_t> &ent, int nwords, uint32_t *out) {
    uint32_t pool[POOL];
    uint32_t hc = INIT_A;
    for (int i = 0; i < POOL; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, hc);
    for (int s = 0; s < POOL; ++s)
        for (int d = 0; d < POOL; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (size_t s = POOL; s < ent.size(); ++s)
        for (int d = 0; d < POOL; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
    uint32_t hb = INIT_B;
    for (int i = 0; i < nwords; ++i) {
        uint32_t v = pool[i % POOL];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> XSHIFT;
        out[i] = v;
    }
}

void pcg64_from_seed(uint64_t seed, uint64_t *st4) {
    std::vector<uint32_t> ent;
    push_int(ent, seed);
    uint32_t w[8];
    seed_seq_words(ent, 8, w);
    uint64_t v[4];
    for (int i = 0; i < 4; ++i) v[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    const u128 inc = (initseq << 1) | 1;
    u128 s = 0;
    s = s * PCG_MULT + inc;
    s += initstate;
    s = s * PCG_MULT + inc;
    st4[0] = (uint64_t)(s >> 64);
    st4[1] = (uint64_t)s;
    st4[2] = (uint64_t)(inc >> 64);
    st4[3] = (uint64_t)inc;
}

}  // namespace

extern "C" int rsc_pcg64_block_states(int count, int width, const uint64_t *keys, const int *nkeys,
                                      uint64_t *seeds_out, uint64_t *states_out) {
    if (count < 0 || width < 1) return -1;
    if (count && (!keys || !nkeys || !states_out)) return -2;
    std::vector<uint32_t> ent;
    for (int i = 0; i < count; ++i) {
        const int nk = nkeys[i];
        if (nk < 1 || nk > width) return -3;
        ent.clear();
        for (int t = 0; t < nk; ++t) push_int(ent, keys[(size_t)i * width + t]);
        uint32_t w[2];
        seed_seq_words(ent, 2, w);
        const uint64_t seed = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
        if (seeds_out) seeds_out[i] = seed;
        pcg64_from_seed(seed, states_out + 4 * (size_t)i);
    }
    return 0;
}

extern "C" int rsc_pcg64_seed_states(int count, const uint64_t *seeds, uint64_t *states_out) {
    if (count < 0) return -1;
    if (count && (!seeds || !states_out)) return -2;
    for (int i = 0; i < count; ++i) pcg64_from_seed(seeds[i], states_out + 4 * (size_t)i);
    return 0;
}
