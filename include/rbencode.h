/*
 * rbencode.h -- native columnar ingest and encoding of text columns (librbgpu.so).
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

/* ---- columnar CSV ingest (rb_csv.cpp): load_relation, relation.py:186-257.
 * rb_csv_parse reads CSV with the semantics of Python's csv.reader default
 * dialect over a file opened with newline=""; the first record is the
 * header.  Status: RB_CSV_OK; RB_CSV_FIELD_COUNT (a record's field count
 * differs from the header's; *err_line = its record number, data records
 * numbered from 2 as in relation.py); RB_CSV_NEEDS_PYTHON (invalid UTF-8, a
 * NUL byte, a field over the csv field limit: run csv.reader for its exact
 * behaviour); RB_CSV_EMPTY (no header row). */
#define RB_CSV_OK 0
#define RB_CSV_FIELD_COUNT (-1)
#define RB_CSV_NEEDS_PYTHON (-2)
#define RB_CSV_EMPTY (-3)
#define RB_CSV_INVALID (-4)
typedef struct rb_csv rb_csv;
int rb_csv_parse(const char* data, int64_t len, rb_csv** out, int64_t* err_line);
int rb_csv_shape(const rb_csv* t, int64_t* rows, int32_t* cols);
int rb_csv_header(const rb_csv* t, int32_t col, const char** bytes, int64_t* nbytes);
/* the cells of one column: bytes [offsets[r], offsets[r+1]) of *bytes, valid until rb_csv_free */
int rb_csv_column(const rb_csv* t, int32_t col, const char** bytes, int64_t* nbytes, const int64_t** offsets);
void rb_csv_free(rb_csv* t);

/* parse_number (relation.py:64-77) per cell: status[i] = 1 number (out[i]),
 * 0 not a number, 2 the cell is not ASCII (decide it in Python) */
void rb_parse_numbers(const char* buf, const int64_t* offsets, int64_t n, double* out, uint8_t* status);
/* len(cell.split()) per cell, -1 when the cell is not ASCII */
void rb_token_counts(const char* buf, const int64_t* offsets, int64_t n, int32_t* counts);

#ifdef __cplusplus
}
#endif
#endif /* RBENCODE_H */
