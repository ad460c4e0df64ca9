/*
 * rbencode.h -- native columnar encoding of ASCII text columns (librbgpu.so).
 *
 * Host-side producers of the device columns of include/rbgpu.h.  Each
 * restates, for all-ASCII columns, the reference's Python encoding:
 *   rb_encode_eq_codes  EncodedRelation.eq_codes     pkg/src/ruleblock/encode.py:77-89
 *   rb_encode_tokens    EncodedRelation.tokens       pkg/src/ruleblock/encode.py:126-138
 *   rb_encode_chars     EncodedRelation.chars        pkg/src/ruleblock/encode.py:140-154
 * Input: one byte buffer with the column's values back to back,
 * offsets[n+1], and an optional missing mask.  The caller routes columns
 * with any non-ASCII value to the Python encoder (exact CPython semantics).
 */
#ifndef RBENCODE_H
#define RBENCODE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* codes[i] = first-appearance dictionary code of strip(value i), -1 if
 * missing; returns the dictionary size */
int rb_encode_eq_codes(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n, int32_t* codes);

/* sorted unique token ids per row (tokenize: casefold, drop ASCII
 * punctuation, split on whitespace; ids interned in first-appearance order).
 * ids needs offsets[n] entries; returns nnz; *vocab_size = distinct tokens */
int64_t rb_encode_tokens(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n,
                         int64_t* out_offsets, int32_t* ids, int32_t* vocab_size);

/* folded characters (strip + casefold) per row; out needs offsets[n] bytes;
 * returns the number of bytes written */
int64_t rb_encode_chars(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n,
                        int64_t* out_offsets, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif /* RBENCODE_H */
