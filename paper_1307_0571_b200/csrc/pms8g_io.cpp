// pms8g_io.cpp — host-side input for the GPU path: sequence files and the
// problem check fused with the 0..sigma-1 encoding the device consumes.
//
// Behaviour follows the reference's reader and Problem::validate (same
// accepted inputs, same exception classes and messages, so the CLI's stderr
// and exit codes match):
//   read_sequences / parse_fasta / parse_plain   src/io.cpp:41-111
//   write_fasta                                   src/io.cpp:113-127
//   Problem::validate                             src/problem.cpp:7-28
// The implementation is our own: the file is read once into a buffer, a
// cursor yields trimmed lines as string_views, and one record builder serves
// both formats; validation walks the sequences once and produces the codes.
#include <cctype>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>

#include "pms8g.hpp"

namespace pms8g {

namespace {

constexpr std::string_view kBlank = " \t\r\n";

std::string_view trim(std::string_view s) {
    const size_t b = s.find_first_not_of(kBlank);
    if (b == std::string_view::npos) return {};
    return s.substr(b, s.find_last_not_of(kBlank) - b + 1);
}

std::string load_file(const std::string& path) {
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
    if (!f) throw std::runtime_error("cannot open " + path);
    std::string buf;
    char block[1 << 16];
    size_t got;
    while ((got = std::fread(block, 1, sizeof block, f.get())) > 0) buf.append(block, got);
    return buf;
}

// Yields the lines of a buffer (without '\n'), counting them from 1.
class LineCursor {
   public:
    explicit LineCursor(std::string_view text) : text_(text) {}
    bool next(std::string_view& line) {
        if (pos_ >= text_.size()) return false;
        const size_t nl = text_.find('\n', pos_);
        const size_t end = nl == std::string_view::npos ? text_.size() : nl;
        line = text_.substr(pos_, end - pos_);
        pos_ = end + 1;
        ++number_;
        return true;
    }
    int number() const { return number_; }

   private:
    std::string_view text_;
    size_t pos_ = 0;
    int number_ = 0;
};

void append_upper(std::string& dst, std::string_view src) {
    dst.reserve(dst.size() + src.size());
    for (const char ch : src) dst.push_back(static_cast<char>(std::toupper(static_cast<unsigned char>(ch))));
}

// "; key=value" -> metadata[key] = value (other comment lines carry nothing)
void take_annotation(std::string_view body, SequenceFile& out) {
    body = trim(body);
    const size_t eq = body.find('=');
    if (eq == std::string_view::npos || eq == 0) return;
    out.metadata[std::string(trim(body.substr(0, eq)))] = std::string(trim(body.substr(eq + 1)));
}

enum class Format { fasta, plain };

SequenceFile parse(std::string_view text, Format fmt) {
    SequenceFile out;
    LineCursor cur(text);
    std::string_view raw;
    bool open_record = false;  // FASTA: a '>' header has been seen
    while (cur.next(raw)) {
        if (!raw.empty() && raw.back() == '\r') raw.remove_suffix(1);
        const std::string_view line = fmt == Format::plain ? trim(raw) : raw;
        if (line.empty()) continue;
        if (line.front() == ';') {
            // plain files take annotations anywhere; FASTA only in its preamble
            if (fmt == Format::plain || !open_record) take_annotation(line.substr(1), out);
            continue;
        }
        if (fmt == Format::plain) {
            out.sequences.emplace_back();
            append_upper(out.sequences.back(), line);
            continue;
        }
        if (line.front() == '>') {
            out.names.emplace_back(trim(line.substr(1)));
            out.sequences.emplace_back();
            open_record = true;
            continue;
        }
        if (!open_record)
            throw std::runtime_error("malformed FASTA: sequence data before any '>' header at line " +
                                     std::to_string(cur.number()));
        append_upper(out.sequences.back(), trim(line));
    }
    if (fmt == Format::plain) {
        if (out.sequences.empty()) throw std::runtime_error("no sequences found");
        return out;
    }
    if (out.sequences.empty()) throw std::runtime_error("malformed FASTA: no records found");
    for (size_t r = 0; r < out.sequences.size(); ++r)
        if (out.sequences[r].empty())
            throw std::runtime_error("malformed FASTA: record " + std::to_string(r + 1) + " (" + out.names[r] +
                                     ") is empty");
    return out;
}

// The first line that is neither blank nor a comment decides the format.
Format sniff(std::string_view text) {
    LineCursor cur(text);
    std::string_view line;
    while (cur.next(line)) {
        line = trim(line);
        if (!line.empty() && line.front() != ';') return line.front() == '>' ? Format::fasta : Format::plain;
    }
    return Format::plain;
}

}  // namespace

SequenceFile read_sequences(const std::string& path) {
    const std::string text = load_file(path);
    return parse(text, sniff(text));
}

SequenceFile read_plain(const std::string& path) { return parse(load_file(path), Format::plain); }

void write_fasta(const std::string& path, const std::vector<std::string>& names,
                 const std::vector<std::string>& sequences,
                 const std::vector<std::pair<std::string, std::string>>& metadata) {
    std::string text;
    for (const auto& kv : metadata) text += "; " + kv.first + "=" + kv.second + "\n";
    constexpr size_t kWidth = 70;  // residues per line
    for (size_t i = 0; i < sequences.size(); ++i) {
        text += '>';
        text += i < names.size() ? names[i] : "seq_" + std::to_string(i);
        text += '\n';
        const std::string& s = sequences[i];
        for (size_t at = 0; at < s.size(); at += kWidth) {
            text.append(s, at, kWidth);
            text += '\n';
        }
    }
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
    if (!f) throw std::runtime_error("cannot write " + path);
    if (std::fwrite(text.data(), 1, text.size(), f.get()) != text.size())
        throw std::runtime_error("write failed for " + path);
}

std::vector<uint8_t> encode_problem(const Problem& p) {
    const int n = p.n();
    if (n == 0) throw std::invalid_argument("no input sequences");
    const int m = p.m(), l = p.motif_length, d = p.max_mismatches;
    if (l < 1) throw std::invalid_argument("motif length must be >= 1");
    if (l > m)
        throw std::invalid_argument("motif length " + std::to_string(l) + " exceeds sequence length " +
                                    std::to_string(m));
    if (d < 0 || d > l)
        throw std::invalid_argument("mismatch budget must be in [0, l], got " + std::to_string(d));
    // symbol -> code lookup (-1: not in the alphabet)
    int code_of[256];
    for (int& c : code_of) c = -1;
    for (size_t c = 0; c < p.alphabet.size(); ++c) code_of[static_cast<unsigned char>(p.alphabet[c])] = static_cast<int>(c);
    std::vector<uint8_t> codes(static_cast<size_t>(n) * m);
    uint8_t* dst = codes.data();
    for (int i = 0; i < n; ++i) {
        const std::string& s = p.sequences[i];
        if (static_cast<int>(s.size()) != m)
            throw std::invalid_argument("sequence " + std::to_string(i) + " has length " + std::to_string(s.size()) +
                                        ", expected " + std::to_string(m));
        for (int j = 0; j < m; ++j) {
            const int c = code_of[static_cast<unsigned char>(s[j])];
            if (c < 0)
                throw std::invalid_argument("sequence " + std::to_string(i) + ", position " + std::to_string(j) +
                                            ": symbol '" + s[j] + "' not in alphabet " + p.alphabet_name);
            *dst++ = static_cast<uint8_t>(c);
        }
    }
    return codes;
}

void Problem::validate() const { (void)encode_problem(*this); }

}  // namespace pms8g
