// rb_csv.cpp -- columnar CSV ingest (the reference's
// load_relation, pkg/src/ruleblock/relation.py:186-257).
//
// The reference reads a relation with Python's csv.reader (default "excel"
// dialect) over a file opened with newline="" and builds one Python object
// per cell and per row (~13 us/tuple).  This tokenizer restates that
// reader's state machine (CPython Modules/_csv.c, parse_process_char, non
// strict, doublequote, no escapechar) over the raw UTF-8 bytes -- every
// structural character is ASCII, so byte-level parsing is exact -- and
// writes the cells column-major: one byte buffer + int64 offsets per column,
// ready for the native encoders (rb_encode.cpp) without per-row objects.
//
// Inputs the Python reader would reject or that need its exact error text
// (invalid UTF-8, a NUL byte, a field longer than the 131072-character field
// limit) return RB_CSV_NEEDS_PYTHON; the caller then runs csv.reader itself.
#include <stdint.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rbencode.h"

struct rb_csv {
    std::vector<std::string> header;
    std::vector<std::string> data;            // per column: cells back to back
    std::vector<std::vector<int64_t>> offs;   // per column: rows + 1 offsets
    int64_t rows = 0;
};

namespace {

bool valid_utf8(const unsigned char* s, int64_t n) {
    int64_t i = 0;
    while (i < n) {
        const unsigned char c = s[i];
        if (c < 0x80) {
            i++;
            continue;
        }
        int len;
        uint32_t cp;
        if ((c & 0xE0) == 0xC0) {
            len = 2;
            cp = c & 0x1F;
        } else if ((c & 0xF0) == 0xE0) {
            len = 3;
            cp = c & 0x0F;
        } else if ((c & 0xF8) == 0xF0) {
            len = 4;
            cp = c & 0x07;
        } else {
            return false;
        }
        if (i + len > n) return false;
        for (int k = 1; k < len; k++) {
            if ((s[i + k] & 0xC0) != 0x80) return false;
            cp = (cp << 6) | (s[i + k] & 0x3F);
        }
        if ((len == 2 && cp < 0x80) || (len == 3 && cp < 0x800) || (len == 4 && cp < 0x10000) || cp > 0x10FFFF ||
            (cp >= 0xD800 && cp <= 0xDFFF))
            return false;
        i += len;
    }
    return true;
}

inline bool py_space(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f); }
inline bool isdig(unsigned char c) { return c >= '0' && c <= '9'; }

enum State { START_RECORD, START_FIELD, IN_FIELD, IN_QUOTED_FIELD, QUOTE_IN_QUOTED_FIELD, EAT_CRNL };
constexpr int64_t FIELD_LIMIT = 131072;  // csv.field_size_limit() default (characters; bytes >= characters)

}  // namespace

extern "C" {

int rb_csv_parse(const char* data, int64_t len, rb_csv** out, int64_t* err_line) {
    if (!out || (!data && len)) return RB_CSV_INVALID;
    *out = nullptr;
    if (err_line) *err_line = 0;
    const unsigned char* s = (const unsigned char*)data;
    if (!valid_utf8(s, len)) return RB_CSV_NEEDS_PYTHON;
    if (len && memchr(data, 0, (size_t)len)) return RB_CSV_NEEDS_PYTHON;

    rb_csv* t = new rb_csv();
    // Fields go straight into their column's buffer (the header's into
    // t->header); a record whose field count differs from the header's is an
    // error, so nothing needs undoing.
    int64_t nfield = 0;     // fields saved in the current record
    int64_t field_len = 0;  // bytes of the current field
    bool have_header = false;
    int64_t record_no = 0;  // 1 = header (relation.py: data lines are numbered from 2)
    State st = START_RECORD;
    int rc = RB_CSV_OK;
    std::string hfield;
    auto cur = [&]() -> std::string* {  // buffer of the field being built; null when beyond the header's width
        if (!have_header) return &hfield;
        return nfield < (int64_t)t->data.size() ? &t->data[nfield] : nullptr;
    };
    auto add = [&](char ch) {
        field_len++;
        if (std::string* b = cur()) b->push_back(ch);
    };
    auto save_field = [&]() {
        if (!have_header) {
            t->header.push_back(hfield);
            hfield.clear();
        } else if (nfield < (int64_t)t->data.size()) {
            t->offs[nfield].push_back((int64_t)t->data[nfield].size());
        }
        nfield++;
        field_len = 0;
    };
    auto emit = [&]() -> bool {  // a complete record; false on a field-count mismatch
        record_no++;
        if (!have_header) {
            t->data.assign(t->header.size(), std::string());
            t->offs.assign(t->header.size(), std::vector<int64_t>(1, 0));
            have_header = true;
        } else {
            if (nfield != (int64_t)t->header.size()) {
                if (err_line) *err_line = record_no;
                rc = RB_CSV_FIELD_COUNT;
                return false;
            }
            t->rows++;
        }
        nfield = 0;
        return true;
    };
    // one event: a byte, or EOL (-1) after each line (newline="": a line ends
    // after \n, after \r\n, after a \r not followed by \n, or at EOF)
    auto process = [&](int c) -> bool {
        const bool eol = c < 0;
        switch (st) {
            case START_RECORD:
                if (eol) return emit();  // an empty line is an empty record
                if (c == '\n' || c == '\r') {
                    st = EAT_CRNL;
                    return true;
                }
                st = START_FIELD;
                [[fallthrough]];
            case START_FIELD:
                if (c == '\n' || c == '\r' || eol) {
                    save_field();
                    st = eol ? START_RECORD : EAT_CRNL;
                    if (eol) return emit();
                } else if (c == '"') {
                    st = IN_QUOTED_FIELD;
                } else if (c == ',') {
                    save_field();
                } else {
                    add((char)c);
                    st = IN_FIELD;
                }
                return true;
            case IN_FIELD:
                if (c == '\n' || c == '\r' || eol) {
                    save_field();
                    st = eol ? START_RECORD : EAT_CRNL;
                    if (eol) return emit();
                } else if (c == ',') {
                    save_field();
                    st = START_FIELD;
                } else {
                    add((char)c);
                }
                return true;
            case IN_QUOTED_FIELD:
                if (eol) return true;
                if (c == '"')
                    st = QUOTE_IN_QUOTED_FIELD;
                else
                    add((char)c);
                return true;
            case QUOTE_IN_QUOTED_FIELD:
                if (c == '"') {
                    add('"');
                    st = IN_QUOTED_FIELD;
                } else if (c == ',') {
                    save_field();
                    st = START_FIELD;
                } else if (c == '\n' || c == '\r' || eol) {
                    save_field();
                    st = eol ? START_RECORD : EAT_CRNL;
                    if (eol) return emit();
                } else {
                    add((char)c);  // not strict: keep the character
                    st = IN_FIELD;
                }
                return true;
            case EAT_CRNL:
                if (c == '\n' || c == '\r') return true;
                if (eol) {
                    st = START_RECORD;
                    return emit();
                }
                rc = RB_CSV_NEEDS_PYTHON;  // cannot happen with newline="" line splitting
                return false;
        }
        return true;
    };

    int64_t i = 0;
    bool ok = true;
    while (ok && i < len) {
        if (st == IN_FIELD) {  // bulk copy of plain field bytes
            int64_t k = i;
            while (k < len && s[k] != ',' && s[k] != '\n' && s[k] != '\r') k++;
            if (k > i) {
                if (std::string* b = cur()) b->append(data + i, (size_t)(k - i));
                field_len += k - i;
                i = k;
                if (field_len > FIELD_LIMIT) {
                    rc = RB_CSV_NEEDS_PYTHON;
                    ok = false;
                }
                continue;
            }
        }
        const int c = s[i++];
        ok = process(c);
        if (ok && field_len > FIELD_LIMIT) {
            rc = RB_CSV_NEEDS_PYTHON;
            ok = false;
        }
        if (ok && (c == '\n' || (c == '\r' && (i >= len || s[i] != '\n')))) ok = process(-1);
    }
    if (ok && len && s[len - 1] != '\n' && s[len - 1] != '\r') ok = process(-1);  // last line without terminator
    // end of input inside a record (csv.reader, not strict): the partial record is kept
    if (ok && (field_len != 0 || st == IN_QUOTED_FIELD)) {
        save_field();
        ok = emit();
    }
    if (!ok) {
        delete t;
        return rc;
    }
    if (!have_header) {
        delete t;
        return RB_CSV_EMPTY;
    }
    *out = t;
    return RB_CSV_OK;
}

int rb_csv_shape(const rb_csv* t, int64_t* rows, int32_t* cols) {
    if (!t || !rows || !cols) return RB_CSV_INVALID;
    *rows = t->rows;
    *cols = (int32_t)t->header.size();
    return RB_CSV_OK;
}

int rb_csv_header(const rb_csv* t, int32_t col, const char** bytes, int64_t* nbytes) {
    if (!t || col < 0 || col >= (int32_t)t->header.size() || !bytes || !nbytes) return RB_CSV_INVALID;
    *bytes = t->header[col].data();
    *nbytes = (int64_t)t->header[col].size();
    return RB_CSV_OK;
}

int rb_csv_column(const rb_csv* t, int32_t col, const char** bytes, int64_t* nbytes, const int64_t** offsets) {
    if (!t || col < 0 || col >= (int32_t)t->data.size() || !bytes || !nbytes || !offsets) return RB_CSV_INVALID;
    *bytes = t->data[col].data();
    *nbytes = (int64_t)t->data[col].size();
    *offsets = t->offs[col].data();
    return RB_CSV_OK;
}

void rb_csv_free(rb_csv* t) { delete t; }

// parse_number (relation.py:64-77) for ASCII cells:
//   text.strip(); drop a leading run of [whitespace $] and trailing
//   whitespace (_CURRENCY_RE; its other glyphs are not ASCII); drop commas
//   followed by exactly three digits and then a non-digit or the end
//   (_THOUSANDS_RE); then float(): [sign] digits [. digits] [e [sign] digits]
//   with single underscores between digits; non-finite values are rejected
//   (inf / nan spellings never parse to a finite value).
void rb_parse_numbers(const char* buf, const int64_t* offsets, int64_t n, double* out, uint8_t* status) {
    std::string clean;
    for (int64_t i = 0; i < n; i++) {
        const unsigned char* b = (const unsigned char*)buf + offsets[i];
        const unsigned char* e = (const unsigned char*)buf + offsets[i + 1];
        out[i] = 0.0;
        bool ascii = true;
        for (const unsigned char* p = b; p < e; p++) ascii &= *p < 0x80;
        if (!ascii) {
            status[i] = 2;
            continue;
        }
        while (b < e && py_space(*b)) b++;  // strip()
        while (e > b && py_space(e[-1])) e--;
        while (b < e && (py_space(*b) || *b == '$')) b++;  // _CURRENCY_RE
        clean.clear();
        for (const unsigned char* p = b; p < e; p++) {
            if (*p == ',' && e - p >= 4 && isdig(p[1]) && isdig(p[2]) && isdig(p[3]) && (e - p == 4 || !isdig(p[4])))
                continue;  // _THOUSANDS_RE
            clean.push_back((char)*p);
        }
        status[i] = 0;
        // float() grammar
        const char* q = clean.c_str();
        const char* qe = q + clean.size();
        std::string num;
        if (q < qe && (*q == '+' || *q == '-')) num.push_back(*q++);
        auto digits = [&](bool& any) -> bool {  // digit (['_'] digit)*; false on a misplaced underscore
            any = false;
            while (q < qe) {
                if (isdig((unsigned char)*q)) {
                    num.push_back(*q++);
                    any = true;
                } else if (*q == '_' && any && q + 1 < qe && isdig((unsigned char)q[1])) {
                    q++;
                } else {
                    break;
                }
            }
            return true;
        };
        bool int_part = false, frac_part = false;
        digits(int_part);
        if (q < qe && *q == '.') {
            num.push_back(*q++);
            digits(frac_part);
        }
        if (!int_part && !frac_part) continue;
        if (q < qe && (*q == 'e' || *q == 'E')) {
            num.push_back(*q++);
            if (q < qe && (*q == '+' || *q == '-')) num.push_back(*q++);
            bool exp_part = false;
            digits(exp_part);
            if (!exp_part) continue;
        }
        if (q != qe) continue;
        const double v = std::strtod(num.c_str(), nullptr);  // correctly rounded, as float()
        if (!std::isfinite(v)) continue;
        out[i] = v;
        status[i] = 1;
    }
}

// len(cell.split()) for ASCII cells (whitespace as str.isspace), -1 otherwise
void rb_token_counts(const char* buf, const int64_t* offsets, int64_t n, int32_t* counts) {
    for (int64_t i = 0; i < n; i++) {
        const unsigned char* b = (const unsigned char*)buf + offsets[i];
        const unsigned char* e = (const unsigned char*)buf + offsets[i + 1];
        int32_t cnt = 0;
        bool in = false, ascii = true;
        for (const unsigned char* p = b; p < e; p++) {
            ascii &= *p < 0x80;
            const bool sp = py_space(*p);
            if (!sp && !in) cnt++;
            in = !sp;
        }
        counts[i] = ascii ? cnt : -1;
    }
}

}  // extern "C"
