// prism-b200 trace synthesis and JSONL I/O. Draw order and rounding follow
// reference proj/src/workload.cpp (cited per function). The reference parses
// with nlohmann::json; here a small strict parser accepts exactly the flat
// objects the trace format uses, and numbers go through strtod (correctly
// rounded, like nlohmann), so parsed TraceEvents are identical.
#include "msim/workload.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>

namespace msim::workload {

namespace {

struct JsonValue {
    enum Kind { kNumber, kString, kBool, kNull } kind = kNull;
    double number = 0.0;
    bool integral = false;
    long long integer = 0;
    std::string text;
};

class LineParser {
public:
    explicit LineParser(const std::string& s) : s_(s) {}

    // Parses one JSON object of scalar members; returns false on syntax error.
    bool object(std::map<std::string, JsonValue>& out) {
        skip();
        if (!eat('{')) return false;
        skip();
        if (eat('}')) return tail();
        while (true) {
            std::string key;
            skip();
            if (!string(key)) return false;
            skip();
            if (!eat(':')) return false;
            skip();
            JsonValue v;
            if (!value(v)) return false;
            out[key] = std::move(v);
            skip();
            if (eat(',')) continue;
            if (eat('}')) return tail();
            return false;
        }
    }

private:
    bool tail() {
        skip();
        return i_ == s_.size();
    }
    void skip() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
    }
    bool eat(char c) {
        if (i_ < s_.size() && s_[i_] == c) {
            ++i_;
            return true;
        }
        return false;
    }
    bool literal(const char* word) {
        const std::size_t n = std::char_traits<char>::length(word);
        if (s_.compare(i_, n, word) != 0) return false;
        i_ += n;
        return true;
    }
    bool string(std::string& out) {
        if (!eat('"')) return false;
        while (i_ < s_.size()) {
            const char c = s_[i_++];
            if (c == '"') return true;
            if (static_cast<unsigned char>(c) < 0x20) return false;
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (i_ >= s_.size()) return false;
            const char e = s_[i_++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    if (i_ + 4 > s_.size()) return false;
                    unsigned cp = 0;
                    for (int k = 0; k < 4; ++k) {
                        const char h = s_[i_++];
                        cp <<= 4;
                        if (h >= '0' && h <= '9') cp |= static_cast<unsigned>(h - '0');
                        else if (h >= 'a' && h <= 'f') cp |= static_cast<unsigned>(h - 'a' + 10);
                        else if (h >= 'A' && h <= 'F') cp |= static_cast<unsigned>(h - 'A' + 10);
                        else return false;
                    }
                    if (cp < 0x80) {
                        out.push_back(static_cast<char>(cp));
                    } else if (cp < 0x800) {
                        out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    } else {
                        out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    }
                    break;
                }
                default: return false;
            }
        }
        return false;
    }
    bool value(JsonValue& v) {
        if (i_ >= s_.size()) return false;
        const char c = s_[i_];
        if (c == '"') {
            v.kind = JsonValue::kString;
            return string(v.text);
        }
        if (literal("true")) {
            v.kind = JsonValue::kBool;
            return true;
        }
        if (literal("false")) {
            v.kind = JsonValue::kBool;
            return true;
        }
        if (literal("null")) {
            v.kind = JsonValue::kNull;
            return true;
        }
        // JSON number grammar: -?(0|[1-9][0-9]*)(\.[0-9]+)?([eE][+-]?[0-9]+)?
        const std::size_t start = i_;
        bool frac = false;
        eat('-');
        if (eat('0')) {
        } else if (i_ < s_.size() && s_[i_] >= '1' && s_[i_] <= '9') {
            while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
        } else {
            return false;
        }
        if (eat('.')) {
            frac = true;
            if (!(i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_])))) return false;
            while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
        }
        if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
            frac = true;
            ++i_;
            if (!eat('+')) eat('-');
            if (!(i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_])))) return false;
            while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
        }
        const std::string tok = s_.substr(start, i_ - start);
        v.kind = JsonValue::kNumber;
        v.number = std::strtod(tok.c_str(), nullptr);
        v.integral = !frac;
        if (v.integral) v.integer = std::strtoll(tok.c_str(), nullptr, 10);
        return true;
    }

    const std::string& s_;
    std::size_t i_ = 0;
};

std::string where(const std::string& origin, std::size_t line) { return origin + ":" + std::to_string(line) + ": "; }

double as_double(const std::map<std::string, JsonValue>& o, const char* key, const std::string& at) {
    const auto it = o.find(key);
    if (it == o.end() || it->second.kind != JsonValue::kNumber) {
        throw ParseError(at + "missing/typed field: " + key);
    }
    return it->second.number;
}

int as_int(const std::map<std::string, JsonValue>& o, const char* key, const std::string& at) {
    const auto it = o.find(key);
    if (it == o.end() || it->second.kind != JsonValue::kNumber) {
        throw ParseError(at + "missing/typed field: " + key);
    }
    return it->second.integral ? static_cast<int>(it->second.integer) : static_cast<int>(it->second.number);
}

TraceEvent parse_record(const std::string& line, const std::string& origin, std::size_t line_no) {  // :16-45
    const std::string at = where(origin, line_no);
    std::map<std::string, JsonValue> obj;
    LineParser p(line);
    if (!p.object(obj)) throw ParseError(at + "bad JSON: cannot parse '" + line + "'");
    TraceEvent ev;
    ev.arrival_s = as_double(obj, "t", at);
    const auto m = obj.find("model");
    if (m == obj.end() || m->second.kind != JsonValue::kString) throw ParseError(at + "missing/typed field: model");
    ev.model_id = m->second.text;
    ev.prompt_tokens = as_int(obj, "prompt", at);
    ev.output_tokens = as_int(obj, "output", at);
    if (!(ev.arrival_s >= 0.0)) throw ParseError(at + "negative arrival time");
    if (ev.model_id.empty()) throw ParseError(at + "empty model id");
    if (ev.prompt_tokens < 1) throw ParseError(at + "prompt_tokens must be >= 1");
    if (ev.output_tokens < 1) throw ParseError(at + "output_tokens must be >= 1");
    return ev;
}

std::string json_number(double x) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), x);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (const char c : s) {
        if (c == '"' || c == '\\') {
            o.push_back('\\');
            o.push_back(c);
        } else if (static_cast<unsigned char>(c) < 0x20) {
            char b[8];
            std::snprintf(b, sizeof(b), "\\u%04x", static_cast<unsigned>(static_cast<unsigned char>(c)));
            o += b;
        } else {
            o.push_back(c);
        }
    }
    return o + "\"";
}

}  // namespace

std::vector<TraceEvent> parse_trace_lines(const std::string& content, const std::string& origin) {  // :49-64
    std::vector<TraceEvent> out;
    std::istringstream in(content);
    std::string line;
    std::size_t n = 0;
    while (std::getline(in, line)) {
        ++n;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        TraceEvent ev = parse_record(line, origin, n);
        if (!out.empty() && ev.arrival_s < out.back().arrival_s) {
            throw ParseError(where(origin, n) + "arrival times out of order");
        }
        out.push_back(std::move(ev));
    }
    return out;
}

std::vector<TraceEvent> parse_trace(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw ParseError("cannot open trace file: " + path);
    std::ostringstream all;
    all << f.rdbuf();
    return parse_trace_lines(all.str(), path);
}

void write_trace(const std::string& path, const std::vector<TraceEvent>& trace) {  // :74-85
    std::ofstream f(path);
    if (!f) throw ParseError("cannot open trace file for writing: " + path);
    // Keys in lexicographic order, compact separators (nlohmann's default dump).
    for (const TraceEvent& e : trace) {
        f << "{\"model\":" << json_string(e.model_id) << ",\"output\":" << e.output_tokens
          << ",\"prompt\":" << e.prompt_tokens << ",\"t\":" << json_number(e.arrival_s) << "}\n";
    }
}

std::vector<TraceEvent> scale_trace(const std::vector<TraceEvent>& trace, int n, std::uint64_t seed,
                                    double jitter_window_s) {  // :87-105
    if (n < 1) throw UsageError("scale_trace: factor must be >= 1");
    if (n == 1) return trace;
    Rng rng(substream_seed(seed, "jitter"));
    std::vector<TraceEvent> out;
    out.reserve(trace.size() * static_cast<std::size_t>(n));
    for (const TraceEvent& e : trace) {
        out.push_back(e);
        for (int k = 1; k < n; ++k) {
            TraceEvent c = e;
            c.arrival_s += rng.uniform01() * jitter_window_s;
            out.push_back(std::move(c));
        }
    }
    std::stable_sort(out.begin(), out.end(),
                     [](const TraceEvent& a, const TraceEvent& b) { return a.arrival_s < b.arrival_s; });
    return out;
}

WorkloadStats compute_stats(const std::vector<TraceEvent>& trace, double idle_threshold_s) {  // :107-163
    if (trace.empty()) throw UsageError("compute_stats: empty trace");
    WorkloadStats st;
    st.idle_threshold_s = idle_threshold_s;
    const double t0 = trace.front().arrival_s;
    double t_end = t0;
    std::map<std::string, std::vector<double>> by_model;
    for (const TraceEvent& e : trace) {
        by_model[e.model_id].push_back(e.arrival_s);
        t_end = std::max(t_end, e.arrival_s);
    }
    st.span_s = t_end - t0;
    const auto bins = static_cast<std::size_t>(std::floor(st.span_s / 60.0)) + 1;
    const double hours = st.span_s / 3600.0;
    for (auto& [model, ts] : by_model) {
        ModelStats ms;
        ms.request_count = ts.size();
        std::vector<double> counts(bins, 0.0);
        for (const double t : ts) {
            auto b = static_cast<std::size_t>(std::floor((t - t0) / 60.0));
            counts[std::min(b, bins - 1)] += 1.0;
        }
        double mean = 0.0;
        for (const double c : counts) mean += c;
        mean /= static_cast<double>(bins);
        if (mean > 0.0) {
            double var = 0.0;
            for (const double c : counts) var += (c - mean) * (c - mean);
            var /= static_cast<double>(bins);
            ms.cv_defined = true;
            ms.cv_req_per_min = std::sqrt(var) / mean;
        }
        if (ts.size() >= 2) {
            ms.idle_defined = true;
            for (std::size_t i = 1; i < ts.size(); ++i) ms.idle_intervals_s.push_back(ts[i] - ts[i - 1]);
            std::vector<double> sorted = ms.idle_intervals_s;
            std::sort(sorted.begin(), sorted.end());
            const std::size_t k = sorted.size();
            ms.median_idle_s = k % 2 ? sorted[k / 2] : 0.5 * (sorted[k / 2 - 1] + sorted[k / 2]);
            for (const double g : ms.idle_intervals_s) ms.idle_over_threshold += g > idle_threshold_s ? 1 : 0;
            if (hours > 0.0) ms.idle_over_threshold_per_hour = static_cast<double>(ms.idle_over_threshold) / hours;
        }
        st.models.emplace(model, std::move(ms));
    }
    return st;
}

std::vector<TraceEvent> synth_trace(const SynthSpec& spec, std::uint64_t seed) {  // :165-191
    std::vector<TraceEvent> out;
    for (const ModelProfile& prof : spec.models) {
        Rng rng(substream_seed(seed, "trace:" + prof.model_id));
        for (const RateSegment& seg : prof.segments) {
            if (seg.rate_per_s < 0.0) throw UsageError("synth_trace: negative rate");
            if (seg.end_s < seg.start_s) throw UsageError("synth_trace: segment ends before it starts");
            if (seg.rate_per_s == 0.0) continue;
            for (double t = seg.start_s;;) {
                t += rng.exponential(seg.rate_per_s);
                if (t >= seg.end_s) break;
                TraceEvent e;
                e.arrival_s = t;
                e.model_id = prof.model_id;
                // Draw order: arrival gap, prompt length, output length.
                const double p = rng.lognormal(prof.prompt_median, prof.prompt_sigma);
                e.prompt_tokens = std::max(1, static_cast<int>(std::lround(p)));
                const double o = rng.lognormal(prof.output_median, prof.output_sigma);
                e.output_tokens = std::max(1, static_cast<int>(std::lround(o)));
                out.push_back(std::move(e));
            }
        }
    }
    std::stable_sort(out.begin(), out.end(),
                     [](const TraceEvent& a, const TraceEvent& b) { return a.arrival_s < b.arrival_s; });
    return out;
}

}  // namespace msim::workload
