// rb_encode.cpp -- native columnar encoding of ASCII text columns
// (the host encoding that feeds the device columns).
//
// Restates, for columns whose every value is ASCII, the Python text
// semantics the reference encodes with (pkg/src/ruleblock/):
//   eq codes   EncodedRelation.eq_codes / _canonical_key    encode.py:33-38, 77-89
//              key = str(v).strip(); codes in first-appearance order; missing -1
//   tokens     EncodedRelation.tokens                        encode.py:126-138
//              tokenize = casefold, drop string.punctuation, split on whitespace
//              (measures.py:29-34); ids interned per attribute in first-appearance
//              order, each row sorted and unique
//   chars      EncodedRelation.chars                         encode.py:140-154
//              fold_text = strip().casefold() (measures.py:25-26)
// For ASCII, CPython's str.isspace / strip / split use exactly
// " \t\n\v\f\r\x1c\x1d\x1e\x1f", casefold is A-Z -> a-z, and
// string.punctuation is the 32 ASCII punctuation characters; the Python
// layer routes any column with a non-ASCII value to the Python encoder.
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "../../include/rbencode.h"

namespace {

inline bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }

inline bool py_punct(unsigned char c) {
    return (c >= 33 && c <= 47) || (c >= 58 && c <= 64) || (c >= 91 && c <= 96) || (c >= 123 && c <= 126);
}

inline unsigned char fold(unsigned char c) { return (c >= 'A' && c <= 'Z') ? (unsigned char)(c + 32) : c; }

inline void strip(const char*& b, const char*& e) {
    while (b < e && py_space((unsigned char)*b)) b++;
    while (e > b && py_space((unsigned char)e[-1])) e--;
}

}  // namespace

extern "C" {

// codes[i] = dictionary code of strip(value i) (first appearance), -1 if missing
int rb_encode_eq_codes(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n, int32_t* codes) {
    std::unordered_map<std::string_view, int32_t> dict;
    dict.reserve((size_t)std::min<int64_t>(n, 1 << 20));
    for (int64_t i = 0; i < n; i++) {
        if (missing && missing[i]) {
            codes[i] = -1;
            continue;
        }
        const char* b = buf + offsets[i];
        const char* e = buf + offsets[i + 1];
        strip(b, e);
        auto it = dict.emplace(std::string_view(b, (size_t)(e - b)), (int32_t)dict.size()).first;
        codes[i] = it->second;
    }
    return (int)dict.size();
}

// Token CSR.  ids must hold offsets[n] entries (an upper bound); returns nnz.
// out_offsets has n+1 entries.  A missing row is an empty row (the caller
// keeps the missing mask).
int64_t rb_encode_tokens(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n,
                         int64_t* out_offsets, int32_t* ids, int32_t* vocab_size) {
    const int64_t total = offsets[n];
    std::string folded;
    folded.resize((size_t)total);
    std::unordered_map<std::string_view, int32_t> dict;
    dict.reserve(1 << 16);
    std::vector<int32_t> row;
    int64_t nnz = 0;
    out_offsets[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        row.clear();
        if (!(missing && missing[i])) {
            // casefold + drop punctuation into the folded buffer, then split
            char* w = &folded[(size_t)offsets[i]];
            char* wb = w;
            for (int64_t k = offsets[i]; k < offsets[i + 1]; k++) {
                const unsigned char c = (unsigned char)buf[k];
                if (!py_punct(c)) *w++ = (char)fold(c);
            }
            const char* p = wb;
            const char* end = w;
            while (p < end) {
                while (p < end && py_space((unsigned char)*p)) p++;
                const char* s = p;
                while (p < end && !py_space((unsigned char)*p)) p++;
                if (p > s) {
                    auto it = dict.emplace(std::string_view(s, (size_t)(p - s)), (int32_t)dict.size()).first;
                    row.push_back(it->second);
                }
            }
            std::sort(row.begin(), row.end());
            row.erase(std::unique(row.begin(), row.end()), row.end());
        }
        if (!row.empty()) std::memcpy(ids + nnz, row.data(), sizeof(int32_t) * row.size());
        nnz += (int64_t)row.size();
        out_offsets[i + 1] = nnz;
    }
    if (vocab_size) *vocab_size = (int32_t)dict.size();
    return nnz;
}

// Folded chars CSR (strip + ASCII casefold).  out must hold offsets[n] bytes.
int64_t rb_encode_chars(const char* buf, const int64_t* offsets, const uint8_t* missing, int64_t n,
                        int64_t* out_offsets, uint8_t* out) {
    int64_t at = 0;
    out_offsets[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        if (!(missing && missing[i])) {
            const char* b = buf + offsets[i];
            const char* e = buf + offsets[i + 1];
            strip(b, e);
            for (; b < e; b++) out[at++] = fold((unsigned char)*b);
        }
        out_offsets[i + 1] = at;
    }
    return at;
}

}  // extern "C"
