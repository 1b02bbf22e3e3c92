// pms8g_json.cpp — pms8g_report_json: the `pms8 solve --format json` document.
//
// The reference builds {"motifs": [...], "report": report_to_json(r)} with
// nlohmann::json and prints it with dump(2) (tools/pms8.cpp:31-60,171-176).
// nlohmann's default object type is an ordered std::map, so keys come out
// sorted; this writer emits the same document byte for byte without the
// dependency: sorted keys, two-space indentation, ", " / ": " separators as
// dump(2) lays them out, and doubles in nlohmann's shortest round-trip form.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "pms8g.h"

namespace {

// One JSON value: a leaf (already rendered) or an object/array of children.
struct Value {
    enum Kind { leaf, object, array } kind = leaf;
    std::string text;                                   // leaf
    std::vector<std::pair<std::string, Value>> fields;  // object (kept sorted by key)
    std::vector<Value> items;                           // array
};

std::string quote(const char* s) {
    std::string o = "\"";
    for (const unsigned char* p = reinterpret_cast<const unsigned char*>(s ? s : ""); *p; ++p) {
        switch (*p) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\b': o += "\\b"; break;
            case '\f': o += "\\f"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (*p < 0x20) {
                    char b[8];
                    std::snprintf(b, sizeof b, "\\u%04x", *p);
                    o += b;
                } else {
                    o += static_cast<char>(*p);
                }
        }
    }
    return o + "\"";
}

// nlohmann's number output for a finite double: the shortest digit string
// that reads back to the same value, placed as fixed notation when the decimal
// point falls within [-3, 15] digits of the first digit, else d.ddde+XX.
std::string number(double v) {
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[40];
    int prec = 0;
    for (prec = 0; prec < 17; ++prec) {
        std::snprintf(buf, sizeof buf, "%.*e", prec, v);
        if (std::strtod(buf, nullptr) == v) break;
    }
    // buf = [-]d[.ddd]e[+-]XX -> digits and decimal exponent
    std::string s(buf);
    std::string sign;
    if (s[0] == '-') {
        sign = "-";
        s.erase(0, 1);
    }
    const size_t e = s.find('e');
    const int exp10 = std::atoi(s.c_str() + e + 1);
    std::string digits;
    for (size_t i = 0; i < e; ++i)
        if (s[i] != '.') digits += s[i];
    while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
    const int k = static_cast<int>(digits.size());
    const int n = exp10 + 1;  // position of the decimal point after the first n digits
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
        out += eb;
    }
    return sign + out;
}

Value leaf(std::string t) {
    Value v;
    v.text = std::move(t);
    return v;
}
Value leaf_int(long long x) { return leaf(std::to_string(x)); }
Value leaf_uint(unsigned long long x) { return leaf(std::to_string(x)); }

Value make_object(std::vector<std::pair<std::string, Value>> f) {
    Value v;
    v.kind = Value::object;
    // insertion sort by key (a handful of fields): std::map order
    for (size_t i = 1; i < f.size(); ++i)
        for (size_t j = i; j > 0 && f[j].first < f[j - 1].first; --j) std::swap(f[j], f[j - 1]);
    v.fields = std::move(f);
    return v;
}

void render(const Value& v, int indent, std::string& out) {
    const std::string pad(static_cast<size_t>(indent + 2), ' ');
    if (v.kind == Value::leaf) {
        out += v.text;
    } else if (v.kind == Value::array) {
        if (v.items.empty()) {
            out += "[]";
            return;
        }
        out += "[\n";
        for (size_t i = 0; i < v.items.size(); ++i) {
            out += pad;
            render(v.items[i], indent + 2, out);
            out += i + 1 < v.items.size() ? ",\n" : "\n";
        }
        out += std::string(static_cast<size_t>(indent), ' ') + "]";
    } else {
        if (v.fields.empty()) {
            out += "{}";
            return;
        }
        out += "{\n";
        for (size_t i = 0; i < v.fields.size(); ++i) {
            out += pad + quote(v.fields[i].first.c_str()) + ": ";
            render(v.fields[i].second, indent + 2, out);
            out += i + 1 < v.fields.size() ? ",\n" : "\n";
        }
        out += std::string(static_cast<size_t>(indent), ' ') + "}";
    }
}

}  // namespace

extern "C" int64_t pms8g_report_json(const pms8g_result* res, const char* alphabet_name, const char* command,
                                     char* out, size_t cap) {
    if (!res) return -1;
    const pms8g_report& r = res->report;
    Value motifs;
    motifs.kind = Value::array;
    for (int64_t i = 0; i < res->count; ++i) {
        const std::string m(res->motifs + i * res->l, static_cast<size_t>(res->l));
        motifs.items.push_back(leaf(quote(m.c_str())));
    }
    const unsigned long long tracked =
        r.pair_matrix_words + r.row_matrix_words + r.row_bookkeeping_words + r.packed_words;
    Value memory = make_object({
        {"pair_matrix_words", leaf_uint(r.pair_matrix_words)},
        {"row_matrix_words", leaf_uint(r.row_matrix_words)},
        {"row_bookkeeping_words", leaf_uint(r.row_bookkeeping_words)},
        {"packed_words", leaf_uint(r.packed_words)},
        {"lookup_table_words", leaf_uint(r.lookup_table_words)},
        {"tracked_total_words", leaf_uint(tracked)},
        {"tracked_total_bytes", leaf_uint(tracked * 8)},
    });
    Value counters = make_object({
        {"stacks_explored", leaf_int(r.stacks_explored)},
        {"neighborhoods", leaf_int(r.neighborhoods)},
        {"neighbors_visited", leaf_int(r.neighbors_visited)},
        {"motifs_emitted", leaf_int(r.motifs_emitted)},
    });
    Value report = make_object({
        {"n", leaf_int(r.n)},
        {"m", leaf_int(r.m)},
        {"l", leaf_int(r.l)},
        {"d", leaf_int(r.d)},
        {"alphabet", leaf(quote(alphabet_name))},
        {"threshold", leaf_int(r.threshold)},
        {"workers", leaf_int(r.gpus)},
        {"subproblems", leaf_int(r.subproblems)},
        {"motif_count", leaf_int(r.motif_count)},
        {"wall_seconds", leaf(number(r.wall_seconds))},
        {"sample_seconds", leaf(number(r.sample_seconds))},
        {"pattern_seconds", leaf(number(r.pattern_seconds))},
        {"memory", std::move(memory)},
        {"counters", std::move(counters)},
        {"command", leaf(quote(command))},
    });
    Value doc = make_object({{"motifs", std::move(motifs)}, {"report", std::move(report)}});
    std::string text;
    render(doc, 0, text);
    if (out && cap > 0) {
        const size_t n = text.size() < cap - 1 ? text.size() : cap - 1;
        std::memcpy(out, text.data(), n);
        out[n] = '\0';
    }
    return static_cast<int64_t>(text.size());
}
