/*
 * neuzip_oracle.h -- CPU restatement of the NeuZip bf16 weight codec.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.  The product path (libnzgpu.so) never links it.
 *
 * Every function restates one reference routine from
 * /root/reference/proj/include/neuzip/ (header-only C++20) in plain C11 and
 * cites the file:line it follows.  Parity of this restatement is pinned
 * against the reference itself (oracle/_ref, compiled from the reference
 * headers by oracle/Makefile) and against the committed fixtures under
 * tests/golden/ (see tests/golden/make_golden.py).
 *
 * Status codes (mirror the reference exception taxonomy, errors.hpp:9-32):
 *    0  ok
 *   -1  std::invalid_argument
 *   -2  FormatError "truncated"       (ans.hpp:232, :246, :323)
 *   -3  FormatError "desynchronization" (ans.hpp:253)
 *   -4  FormatError "length / count mismatch" (tensorstore.hpp:116, :219, :226; ans.hpp:344)
 *   -5  NonFiniteError                (tensorstore.hpp:155)
 *   -6  FormatError "table does not sum to 4096" (ans.hpp:100)
 */
#ifndef NEUZIP_ORACLE_H
#define NEUZIP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_OK 0
#define ORC_INVALID_ARGUMENT (-1)
#define ORC_TRUNCATED (-2)
#define ORC_DESYNC (-3)
#define ORC_LENGTH (-4)
#define ORC_NONFINITE (-5)
#define ORC_BAD_TABLE (-6)

/* ans.hpp:30-34 */
#define ORC_PROB_BITS 12u
#define ORC_PROB_SCALE 4096u
#define ORC_STATE_LOW (1u << 23)
#define ORC_CHUNK_SYMBOLS 65536u
#define ORC_TABLE_BYTES 512u

/* ---- bitfloat.hpp ---------------------------------------------------- */
uint16_t orc_bf16_from_float(float f);                        /* bitfloat.hpp:25-32 */
void orc_split(const uint16_t* v, uint64_t n, uint8_t* exponents,
               uint8_t* signmant);                            /* bitfloat.hpp:56-62, tensorstore.hpp:97-102 */
void orc_merge(const uint8_t* exponents, const uint8_t* signmant,
               uint64_t n, uint16_t* out);                    /* bitfloat.hpp:64-71, tensorstore.hpp:119-123 */
int orc_round_mantissa(int m, int k, int* mantissa, int* carry); /* bitfloat.hpp:82-98 */
int orc_truncate_mantissa(int m, int k);                       /* bitfloat.hpp:102-105 */
uint64_t orc_packed_bytes(uint64_t n, int k);
int orc_pack_signed_mantissas(const uint8_t* signs, const uint8_t* mants,
                              uint64_t n, int k, uint8_t* out); /* bitfloat.hpp:124-143 */
int orc_unpack_signed_mantissas(const uint8_t* bytes, uint64_t nbytes, int k,
                                uint64_t n, uint8_t* signs,
                                uint8_t* mants);              /* bitfloat.hpp:145-164 */

/* ---- ans.hpp ---------------------------------------------------------- */
int orc_build_table(const uint64_t* counts, uint16_t* freqs); /* ans.hpp:52-93, :154-156 */
int orc_check_table(const uint16_t* freqs);                    /* ans.hpp:96-103 */
/* Worst-case payload bytes of one chunk of nsym symbols (<= 2 B/symbol + state). */
uint64_t orc_chunk_payload_bound(uint64_t nsym);
/* Returns payload length (>= 4) or a negative status.  ans.hpp:202-225 */
int64_t orc_ans_encode_chunk(const uint8_t* symbols, uint64_t nsym,
                             const uint16_t* freqs, uint8_t* payload);
/* ans.hpp:229-256 */
int orc_ans_decode_chunk(const uint8_t* payload, uint64_t len, uint64_t nsym,
                         const uint16_t* freqs, uint8_t* out);
/* Serialized stream = [u32 nchunks][u32 nsym][u32 len][payload]... (ans.hpp:306-316)
 * of ans_encode (ans.hpp:260-271) with chunk size `chunk_symbols` (65536 in
 * the reference; other sizes compose ans_encode_chunk over S-spans).       */
uint64_t orc_stream_bound(uint64_t n, uint64_t chunk_symbols);
int64_t orc_ans_encode_stream(const uint8_t* symbols, uint64_t n,
                              uint64_t chunk_symbols, const uint16_t* freqs,
                              uint8_t* stream);
/* deserialize_stream (ans.hpp:318-347) + ans_decode (ans.hpp:273-293). */
int orc_ans_decode_stream(const uint8_t* stream, uint64_t len,
                          const uint16_t* freqs, uint8_t* out, uint64_t n);
/* Number of symbols a serialized stream claims (framing walk), or negative. */
int64_t orc_stream_symbol_count(const uint8_t* stream, uint64_t len);

/* ---- tensorstore.hpp -------------------------------------------------- */
/* compress_lossless (tensorstore.hpp:87-106): returns stream length. */
int64_t orc_compress_lossless(const uint16_t* values, uint64_t n,
                              uint64_t chunk_symbols, uint16_t* freqs,
                              uint8_t* stream, uint8_t* signmant);
/* decompress_lossless (tensorstore.hpp:112-125) */
int orc_decompress_lossless(const uint8_t* stream, uint64_t stream_len,
                            const uint16_t* freqs, const uint8_t* signmant,
                            uint64_t signmant_len, uint64_t n, uint16_t* out);
/* compress_lossy (tensorstore.hpp:141-208): returns stream length. */
int64_t orc_compress_lossy(const uint16_t* values, uint64_t n, int k,
                           uint32_t block_size, uint64_t chunk_symbols,
                           uint16_t* freqs, uint8_t* scales, uint8_t* stream,
                           uint8_t* packed);
/* decompress_lossy (tensorstore.hpp:215-238) */
int orc_decompress_lossy(const uint8_t* stream, uint64_t stream_len,
                         const uint16_t* freqs, const uint8_t* packed,
                         uint64_t packed_len, const uint8_t* scales,
                         uint64_t scales_len, int k, uint32_t block_size,
                         uint64_t n, uint16_t* out);
/* Element-wise lossy round trip of one value (oracles.hpp:129-153 / tensorstore.hpp:179-198, :229-236). */
uint16_t orc_lossy_roundtrip(uint16_t bits, uint8_t scale_byte, int k);
void orc_lossy_roundtrip_many(const uint16_t* bits, const uint8_t* scales, uint64_t n, int k,
                              uint16_t* out);
/* footprint().total() (tensorstore.hpp:242-283) */
uint64_t orc_footprint_total(uint64_t stream_len, uint64_t mantissa_bytes,
                             uint64_t scale_bytes, uint64_t ndim);

/* ---- rng.hpp (synthetic inputs) and crc32.hpp ------------------------- */
uint64_t orc_rng_word(uint64_t seed, uint64_t counter);        /* rng.hpp:30-32 */
uint64_t orc_rng_derive(uint64_t seed, uint64_t tag);          /* rng.hpp:35-37 */
double orc_rng_uniform(uint64_t seed, uint64_t counter);       /* rng.hpp:40-42 */
double orc_rng_gaussian(uint64_t seed, uint64_t index);        /* rng.hpp:45-51 */
void orc_gaussian_bf16_range(uint64_t seed, uint64_t start, uint64_t n, double sigma,
                             uint16_t* out);   /* rng.hpp:73-81, samples [start, start+n) */
void orc_gaussian_bf16(uint64_t seed, uint64_t n, double sigma,
                       uint16_t* out);                        /* rng.hpp:73-81 */
uint32_t orc_crc32(const uint8_t* data, uint64_t n);           /* crc32.hpp:26-43 */

#ifdef __cplusplus
}
#endif

#endif
