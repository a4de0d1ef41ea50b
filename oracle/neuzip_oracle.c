/*
 * neuzip_oracle.c -- CPU restatement of the NeuZip bf16 weight codec.
 *
 * TEST INFRASTRUCTURE ONLY (see neuzip_oracle.h).  Plain, scalar,
 * single-threaded C11 that follows the reference line by line; clarity over
 * speed.  Reference paths are relative to /root/reference/proj/include/neuzip/.
 */
#include "neuzip_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* bitfloat.hpp                                                             */
/* ------------------------------------------------------------------------ */

/* bitfloat.hpp:25-32 -- RNE float -> bf16, NaN quietened with |0x40. */
uint16_t orc_bf16_from_float(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x0040u);
    uint32_t rounded = u + 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(rounded >> 16);
}

/* bitfloat.hpp:35-37 */
static double bf16_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* bitfloat.hpp:56-62 + tensorstore.hpp:97-102: exponent plane and the
 * sign+mantissa byte (s << 7) | m. */
void orc_split(const uint16_t* v, uint64_t n, uint8_t* exponents, uint8_t* signmant) {
    for (uint64_t i = 0; i < n; ++i) {
        uint16_t b = v[i];
        uint8_t s = (uint8_t)(b >> 15);
        uint8_t e = (uint8_t)((b >> 7) & 0xFFu);
        uint8_t m = (uint8_t)(b & 0x7Fu);
        if (exponents) exponents[i] = e;
        if (signmant) signmant[i] = (uint8_t)((s << 7) | m);
    }
}

/* bitfloat.hpp:64-71 with the tensorstore.hpp:119-123 field unpacking. */
void orc_merge(const uint8_t* exponents, const uint8_t* signmant, uint64_t n, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        uint16_t s = (uint16_t)(signmant[i] >> 7);
        uint16_t m = (uint16_t)(signmant[i] & 0x7Fu);
        out[i] = (uint16_t)((s << 15) | ((uint16_t)exponents[i] << 7) | m);
    }
}

/* bitfloat.hpp:82-98 -- RNE to k retained bits; carry when kept >= 2^k. */
int orc_round_mantissa(int m, int k, int* mantissa, int* carry) {
    if (k != 0 && k != 1 && k != 3) return ORC_INVALID_ARGUMENT;
    if (m < 0 || m > 127) return ORC_INVALID_ARGUMENT;
    int drop = 7 - k;
    int rem = m & ((1 << drop) - 1);
    int half = 1 << (drop - 1);
    int kept = m >> drop;
    if (rem > half || (rem == half && (kept & 1))) kept += 1;
    if (kept >= (1 << k)) {
        *mantissa = 0;
        *carry = 1;
    } else {
        *mantissa = kept << drop;
        *carry = 0;
    }
    return ORC_OK;
}

/* bitfloat.hpp:102-105 */
int orc_truncate_mantissa(int m, int k) {
    int drop = 7 - k;
    return (m >> drop) << drop;
}

static int valid_pack_precision(int k) { return k == 0 || k == 1 || k == 3 || k == 7; }

uint64_t orc_packed_bytes(uint64_t n, int k) { return (n * (uint64_t)(k + 1) + 7) / 8; }

/* bitfloat.hpp:124-143 -- MSB-first (k+1)-bit items, zero-padded tail. */
int orc_pack_signed_mantissas(const uint8_t* signs, const uint8_t* mants, uint64_t n, int k,
                              uint8_t* out) {
    if (!valid_pack_precision(k)) return ORC_INVALID_ARGUMENT;
    unsigned width = (unsigned)k + 1;
    uint64_t nbytes = orc_packed_bytes(n, k);
    memset(out, 0, nbytes);
    for (uint64_t i = 0; i < n; ++i) {
        if (signs[i] > 1 || mants[i] >= (1u << k)) return ORC_INVALID_ARGUMENT;
        unsigned value = ((unsigned)signs[i] << k) | mants[i];
        uint64_t bit = i * width;
        unsigned shift = 8 - width - (unsigned)(bit % 8);
        out[bit / 8] |= (uint8_t)(value << shift);
    }
    return ORC_OK;
}

/* bitfloat.hpp:145-164 */
int orc_unpack_signed_mantissas(const uint8_t* bytes, uint64_t nbytes, int k, uint64_t n,
                                uint8_t* signs, uint8_t* mants) {
    if (!valid_pack_precision(k)) return ORC_INVALID_ARGUMENT;
    unsigned width = (unsigned)k + 1;
    if (nbytes != orc_packed_bytes(n, k)) return ORC_INVALID_ARGUMENT;
    unsigned mask = (1u << width) - 1u;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t bit = i * width;
        unsigned shift = 8 - width - (unsigned)(bit % 8);
        unsigned value = ((unsigned)bytes[bit / 8] >> shift) & mask;
        signs[i] = (uint8_t)(value >> k);
        mants[i] = (uint8_t)(value & ((1u << k) - 1u));
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ans.hpp                                                                  */
/* ------------------------------------------------------------------------ */

/* FrequencyTable::from_counts, ans.hpp:52-93.
 * 1. floor(c * 4096 / T) with remainders (ans.hpp:62-70)
 * 2. stable sort of symbol indices by remainder, descending (ans.hpp:72-76);
 *    restated as a stable insertion sort
 * 3. +1 to the first `deficit` entries of that order (ans.hpp:77-80)
 * 4. floor-at-1 repair, donor = first argmax of freqs (ans.hpp:83-91)   */
int orc_build_table(const uint64_t* counts, uint16_t* freqs) {
    uint64_t total = 0;
    for (int s = 0; s < 256; ++s) total += counts[s];
    if (total == 0) return ORC_INVALID_ARGUMENT;

    uint64_t rem[256];
    uint32_t assigned = 0;
    for (int s = 0; s < 256; ++s) {
        uint64_t scaled = counts[s] * (uint64_t)ORC_PROB_SCALE;
        freqs[s] = (uint16_t)(scaled / total);
        rem[s] = scaled % total;
        assigned += freqs[s];
    }
    int order[256];
    for (int i = 0; i < 256; ++i) {
        /* stable insertion: move past every earlier element with rem >= rem[i] */
        int j = i;
        while (j > 0 && rem[order[j - 1]] < rem[i]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = i;
    }
    for (int i = 0; assigned < ORC_PROB_SCALE; ++i) {
        ++freqs[order[i % 256]];
        ++assigned;
    }
    for (int s = 0; s < 256; ++s) {
        if (counts[s] == 0 || freqs[s] != 0) continue;
        int donor = 0;
        for (int d = 1; d < 256; ++d)
            if (freqs[d] > freqs[donor]) donor = d;
        --freqs[donor];
        freqs[s] = 1;
    }
    return ORC_OK;
}

/* FrequencyTable::from_frequencies, ans.hpp:96-103 */
int orc_check_table(const uint16_t* freqs) {
    uint32_t sum = 0;
    for (int s = 0; s < 256; ++s) sum += freqs[s];
    return sum == ORC_PROB_SCALE ? ORC_OK : ORC_BAD_TABLE;
}

/* FrequencyTable ctor, ans.hpp:137-147: cumulative starts + slot LUT. */
static void table_tables(const uint16_t* freqs, uint32_t* cum, uint8_t* slot_to_symbol) {
    uint32_t c = 0;
    for (int s = 0; s < 256; ++s) {
        cum[s] = c;
        if (slot_to_symbol)
            for (uint32_t slot = 0; slot < freqs[s]; ++slot) slot_to_symbol[c + slot] = (uint8_t)s;
        c += freqs[s];
    }
}

uint64_t orc_chunk_payload_bound(uint64_t nsym) { return 2 * nsym + 4; }

static void put_u32le(uint8_t* p, uint32_t v) { /* ans.hpp:185-190 */
    p[0] = (uint8_t)(v & 0xFFu);
    p[1] = (uint8_t)((v >> 8) & 0xFFu);
    p[2] = (uint8_t)((v >> 16) & 0xFFu);
    p[3] = (uint8_t)(v >> 24);
}

static uint32_t get_u32le(const uint8_t* b) { /* ans.hpp:192-197 */
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

/* ans_encode_chunk, ans.hpp:202-225: reverse-order encode; renorm bytes are
 * emitted in reverse consumption order, reversed, then LE32(final state). */
int64_t orc_ans_encode_chunk(const uint8_t* symbols, uint64_t nsym, const uint16_t* freqs,
                             uint8_t* payload) {
    uint32_t cum[256];
    table_tables(freqs, cum, NULL);
    uint32_t state = ORC_STATE_LOW;
    uint64_t nb = 0;
    for (uint64_t i = nsym; i-- > 0;) {
        uint8_t s = symbols[i];
        uint32_t f = freqs[s];
        if (f == 0) return ORC_INVALID_ARGUMENT;
        uint32_t limit = f << 19;
        while (state >= limit) {
            payload[nb++] = (uint8_t)(state & 0xFFu);
            state >>= 8;
        }
        state = ((state / f) << ORC_PROB_BITS) + (state % f) + cum[s];
    }
    for (uint64_t a = 0, b = nb; a + 1 < b; ++a, --b) {
        uint8_t t = payload[a];
        payload[a] = payload[b - 1];
        payload[b - 1] = t;
    }
    put_u32le(payload + nb, state);
    return (int64_t)(nb + 4);
}

/* ans_decode_chunk, ans.hpp:229-256 */
int orc_ans_decode_chunk(const uint8_t* payload, uint64_t len, uint64_t nsym,
                         const uint16_t* freqs, uint8_t* out) {
    if (len < 4) return ORC_TRUNCATED;
    uint32_t cum[256];
    uint8_t* lut = (uint8_t*)malloc(ORC_PROB_SCALE);
    table_tables(freqs, cum, lut);
    uint64_t limit = len - 4;
    uint32_t state = get_u32le(payload + limit);
    uint64_t pos = 0;
    int rc = ORC_OK;
    for (uint64_t i = 0; i < nsym; ++i) {
        uint32_t slot = state & (ORC_PROB_SCALE - 1);
        uint8_t s = lut[slot];
        state = (uint32_t)freqs[s] * (state >> ORC_PROB_BITS) + slot - cum[s];
        while (state < ORC_STATE_LOW) {
            if (pos >= limit) {
                rc = ORC_TRUNCATED;
                goto done;
            }
            state = (state << 8) | payload[pos++];
        }
        out[i] = s;
    }
    if (state != ORC_STATE_LOW || pos != limit) rc = ORC_DESYNC;
done:
    free(lut);
    return rc;
}

uint64_t orc_stream_bound(uint64_t n, uint64_t chunk_symbols) {
    uint64_t chunks = (n + chunk_symbols - 1) / chunk_symbols;
    return 4 + chunks * 8 + 2 * n + 4 * chunks;
}

/* ans_encode (ans.hpp:260-271) then serialize_stream (ans.hpp:306-316). */
int64_t orc_ans_encode_stream(const uint8_t* symbols, uint64_t n, uint64_t chunk_symbols,
                              const uint16_t* freqs, uint8_t* stream) {
    if (chunk_symbols == 0) return ORC_INVALID_ARGUMENT;
    uint64_t chunks = (n + chunk_symbols - 1) / chunk_symbols;
    put_u32le(stream, (uint32_t)chunks);
    uint64_t pos = 4;
    for (uint64_t c = 0; c < chunks; ++c) {
        uint64_t begin = c * chunk_symbols;
        uint64_t len = n - begin < chunk_symbols ? n - begin : chunk_symbols;
        int64_t plen = orc_ans_encode_chunk(symbols + begin, len, freqs, stream + pos + 8);
        if (plen < 0) return plen;
        put_u32le(stream + pos, (uint32_t)len);
        put_u32le(stream + pos + 4, (uint32_t)plen);
        pos += 8 + (uint64_t)plen;
    }
    return (int64_t)pos;
}

/* deserialize_stream framing walk (ans.hpp:318-347). */
int64_t orc_stream_symbol_count(const uint8_t* stream, uint64_t len) {
    if (len < 4) return ORC_TRUNCATED;
    uint32_t chunks = get_u32le(stream);
    uint64_t pos = 4, total = 0;
    for (uint32_t c = 0; c < chunks; ++c) {
        if (len - pos < 8) return ORC_TRUNCATED;
        total += get_u32le(stream + pos);
        uint32_t plen = get_u32le(stream + pos + 4);
        pos += 8;
        if (len - pos < plen) return ORC_TRUNCATED;
        pos += plen;
    }
    if (pos != len) return ORC_LENGTH; /* "ans stream: trailing bytes" */
    return (int64_t)total;
}

/* deserialize_stream (ans.hpp:318-347) + ans_decode (ans.hpp:273-293).
 * `n` is the capacity of `out`; a stream claiming more symbols is a length
 * mismatch (the caller's tensorstore.hpp:115 check). */
int orc_ans_decode_stream(const uint8_t* stream, uint64_t len, const uint16_t* freqs,
                          uint8_t* out, uint64_t n) {
    int rc = orc_check_table(freqs);
    if (rc) return rc;
    int64_t total = orc_stream_symbol_count(stream, len);
    if (total < 0) return (int)total;
    if ((uint64_t)total != n) return ORC_LENGTH;
    uint32_t chunks = get_u32le(stream);
    uint64_t pos = 4, off = 0;
    for (uint32_t c = 0; c < chunks; ++c) {
        uint32_t nsym = get_u32le(stream + pos);
        uint32_t plen = get_u32le(stream + pos + 4);
        pos += 8;
        rc = orc_ans_decode_chunk(stream + pos, plen, nsym, freqs, out + off);
        if (rc) return rc;
        pos += plen;
        off += nsym;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* tensorstore.hpp                                                          */
/* ------------------------------------------------------------------------ */

/* compress_lossless, tensorstore.hpp:87-106 */
int64_t orc_compress_lossless(const uint16_t* values, uint64_t n, uint64_t chunk_symbols,
                              uint16_t* freqs, uint8_t* stream, uint8_t* signmant) {
    if (n == 0) return ORC_INVALID_ARGUMENT; /* TensorMeta::validate, tensorstore.hpp:47-53 */
    uint8_t* exps = (uint8_t*)malloc(n);
    uint64_t counts[256] = {0};
    orc_split(values, n, exps, signmant);
    for (uint64_t i = 0; i < n; ++i) ++counts[exps[i]];
    int rc = orc_build_table(counts, freqs);
    int64_t len = rc ? rc : orc_ans_encode_stream(exps, n, chunk_symbols, freqs, stream);
    free(exps);
    return len;
}

/* decompress_lossless, tensorstore.hpp:112-125 */
int orc_decompress_lossless(const uint8_t* stream, uint64_t stream_len, const uint16_t* freqs,
                            const uint8_t* signmant, uint64_t signmant_len, uint64_t n,
                            uint16_t* out) {
    int64_t total = orc_stream_symbol_count(stream, stream_len);
    if (total < 0) return (int)total;
    uint8_t* exps = (uint8_t*)malloc(total ? (size_t)total : 1);
    int rc = orc_ans_decode_stream(stream, stream_len, freqs, exps, (uint64_t)total);
    if (rc == ORC_OK && ((uint64_t)total != n || signmant_len != n)) rc = ORC_LENGTH;
    if (rc == ORC_OK) orc_merge(exps, signmant, n, out);
    free(exps);
    return rc;
}

/* detail::scale_coefficient, tensorstore.hpp:135-137 */
static double scale_coefficient(uint8_t scale_byte) { return 1.0 + (double)scale_byte / 128.0; }

/* Per-element lossy normalisation + rounding, tensorstore.hpp:179-198. */
static void lossy_element(uint16_t bits, double c, int k, uint8_t* exponent, uint8_t* sign,
                          uint8_t* item_mant) {
    uint16_t nb = orc_bf16_from_float((float)(bf16_to_double(bits) / c));
    int s = nb >> 15, e = (nb >> 7) & 0xFF, m = nb & 0x7F;
    int rm, carry;
    orc_round_mantissa(m, k, &rm, &carry);
    if (carry) {
        if (e == 254) {
            m = orc_truncate_mantissa(m, k);
        } else {
            e += 1;
            m = 0;
        }
    } else {
        m = rm;
    }
    *exponent = (uint8_t)e;
    *sign = (uint8_t)s;
    *item_mant = (uint8_t)(m >> (7 - k));
}

/* decompress_lossy element, tensorstore.hpp:229-236 */
static uint16_t lossy_rebuild(uint8_t sign, uint8_t exponent, uint8_t mant, int k, double c) {
    uint16_t normalized =
        (uint16_t)(((uint16_t)sign << 15) | ((uint16_t)exponent << 7) | (uint16_t)(mant << (7 - k)));
    return orc_bf16_from_float((float)(bf16_to_double(normalized) * c));
}

uint16_t orc_lossy_roundtrip(uint16_t bits, uint8_t scale_byte, int k) {
    double c = scale_coefficient(scale_byte);
    uint8_t e, s, m;
    lossy_element(bits, c, k, &e, &s, &m);
    return lossy_rebuild(s, e, m, k, c);
}

/* compress_lossy, tensorstore.hpp:141-208 */
int64_t orc_compress_lossy(const uint16_t* values, uint64_t n, int k, uint32_t block_size,
                           uint64_t chunk_symbols, uint16_t* freqs, uint8_t* scales,
                           uint8_t* stream, uint8_t* packed) {
    if (k != 0 && k != 1 && k != 3) return ORC_INVALID_ARGUMENT;
    if (block_size == 0) return ORC_INVALID_ARGUMENT;
    if (n == 0) return ORC_INVALID_ARGUMENT;
    for (uint64_t i = 0; i < n; ++i)
        if ((values[i] & 0x7F80u) == 0x7F80u) return ORC_NONFINITE; /* bitfloat.hpp:41 */
    uint64_t blocks = (n + block_size - 1) / block_size;
    uint8_t* exps = (uint8_t*)malloc(n);
    uint8_t* signs = (uint8_t*)malloc(n);
    uint8_t* mants = (uint8_t*)malloc(n);
    for (uint64_t b = 0; b < blocks; ++b) {
        uint64_t begin = b * block_size;
        uint64_t end = begin + block_size < n ? begin + block_size : n;
        uint64_t max_at = begin;
        for (uint64_t i = begin + 1; i < end; ++i) /* tensorstore.hpp:168-174, strict > */
            if ((values[i] & 0x7FFFu) > (values[max_at] & 0x7FFFu)) max_at = i;
        uint8_t scale_byte = (uint8_t)(values[max_at] & 0x7Fu);
        scales[b] = scale_byte;
        double c = scale_coefficient(scale_byte);
        for (uint64_t i = begin; i < end; ++i) lossy_element(values[i], c, k, &exps[i], &signs[i], &mants[i]);
    }
    uint64_t counts[256] = {0};
    for (uint64_t i = 0; i < n; ++i) ++counts[exps[i]]; /* tensorstore.hpp:201-203 */
    int64_t len = orc_build_table(counts, freqs);
    if (len == 0) len = orc_ans_encode_stream(exps, n, chunk_symbols, freqs, stream);
    if (len >= 0) {
        int rc = orc_pack_signed_mantissas(signs, mants, n, k, packed);
        if (rc) len = rc;
    }
    free(exps);
    free(signs);
    free(mants);
    return len;
}

/* decompress_lossy, tensorstore.hpp:215-238 */
int orc_decompress_lossy(const uint8_t* stream, uint64_t stream_len, const uint16_t* freqs,
                         const uint8_t* packed, uint64_t packed_len, const uint8_t* scales,
                         uint64_t scales_len, int k, uint32_t block_size, uint64_t n,
                         uint16_t* out) {
    if (block_size == 0) return ORC_INVALID_ARGUMENT;
    int64_t total = orc_stream_symbol_count(stream, stream_len);
    if (total < 0) return (int)total;
    if ((uint64_t)total != n) return ORC_LENGTH;
    uint8_t* exps = (uint8_t*)malloc(n ? n : 1);
    uint8_t* signs = (uint8_t*)malloc(n ? n : 1);
    uint8_t* mants = (uint8_t*)malloc(n ? n : 1);
    int rc = orc_ans_decode_stream(stream, stream_len, freqs, exps, n);
    if (rc == ORC_OK) rc = orc_unpack_signed_mantissas(packed, packed_len, k, n, signs, mants);
    if (rc == ORC_OK && scales_len != (n + block_size - 1) / block_size) rc = ORC_LENGTH;
    if (rc == ORC_OK)
        for (uint64_t i = 0; i < n; ++i)
            out[i] = lossy_rebuild(signs[i], exps[i], mants[i], k,
                                   scale_coefficient(scales[i / block_size]));
    free(exps);
    free(signs);
    free(mants);
    return rc;
}

/* footprint(), tensorstore.hpp:242-283; nzt_header_bytes :259-261 */
uint64_t orc_footprint_total(uint64_t stream_len, uint64_t mantissa_bytes, uint64_t scale_bytes,
                             uint64_t ndim) {
    uint64_t header = 4 + 1 + 1 + 4 + 1 + 8 * ndim + 4 + 8 + 8 + 4;
    return stream_len + mantissa_bytes + scale_bytes + ORC_TABLE_BYTES + header;
}

/* ------------------------------------------------------------------------ */
/* rng.hpp / crc32.hpp                                                      */
/* ------------------------------------------------------------------------ */

#define ORC_GOLDEN 0x9E3779B97F4A7C15ull

static uint64_t mix64(uint64_t z) { /* rng.hpp:21-28 */
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

uint64_t orc_rng_word(uint64_t seed, uint64_t counter) { return mix64(seed + (counter + 1) * ORC_GOLDEN); }

uint64_t orc_rng_derive(uint64_t seed, uint64_t tag) { return mix64(seed ^ mix64(tag + ORC_GOLDEN)); }

double orc_rng_uniform(uint64_t seed, uint64_t counter) {
    return (double)(orc_rng_word(seed, counter) >> 11) * 0x1.0p-53;
}

double orc_rng_gaussian(uint64_t seed, uint64_t index) {
    double u1 = ((double)(orc_rng_word(seed, 2 * index) >> 11) + 1.0) * 0x1.0p-53;
    double u2 = orc_rng_uniform(seed, 2 * index + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

/* Samples [start, start + n) of rng::gaussian_bf16 (rng.hpp:73-81): the
 * generator is counter-based, so disjoint ranges can be filled in parallel. */
void orc_gaussian_bf16_range(uint64_t seed, uint64_t start, uint64_t n, double sigma, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = orc_bf16_from_float((float)(sigma * orc_rng_gaussian(seed, start + i)));
}

void orc_gaussian_bf16(uint64_t seed, uint64_t n, double sigma, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_bf16_from_float((float)(sigma * orc_rng_gaussian(seed, i)));
}

uint32_t orc_crc32(const uint8_t* data, uint64_t n) { /* crc32.hpp:12-43 */
    static uint32_t table[256];
    static int init = 0;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int bit = 0; bit < 8; ++bit) c = (c & 1u) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
            table[i] = c;
        }
        init = 1;
    }
    uint32_t state = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n; ++i) state = table[(state ^ data[i]) & 0xFFu] ^ (state >> 8);
    return state ^ 0xFFFFFFFFu;
}

/* Vectorised form of orc_lossy_roundtrip for the exhaustive parity sweep. */
void orc_lossy_roundtrip_many(const uint16_t* bits, const uint8_t* scales, uint64_t n, int k, uint16_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_lossy_roundtrip(bits[i], scales[i], k);
}
