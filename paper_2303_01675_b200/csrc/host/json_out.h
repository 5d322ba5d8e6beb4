// Minimal deterministic JSON writer for plans, timelines and tuning logs.
// Doubles are printed with %.17g so artifacts round-trip bit-exactly.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace pipetune {
namespace json {

class Writer {
  public:
    std::string out;

    Writer& raw(const std::string& s) {
        out += s;
        return *this;
    }
    Writer& str(const std::string& s) {
        out.push_back('"');
        for (char c : s) {
            if (c == '"' || c == '\\') {
                out.push_back('\\');
                out.push_back(c);
            } else if (c == '\n') {
                out += "\\n";
            } else {
                out.push_back(c);
            }
        }
        out.push_back('"');
        return *this;
    }
    Writer& num(long long v) {
        out += std::to_string(v);
        return *this;
    }
    Writer& dbl(double v) {
        char buf[40];
        std::snprintf(buf, sizeof buf, "%.17g", v);
        out += buf;
        return *this;
    }
    Writer& key(const char* k) {
        comma();
        str(k);
        out.push_back(':');
        return *this;
    }
    Writer& begin_obj() {
        comma();
        out.push_back('{');
        return *this;
    }
    Writer& end_obj() {
        out.push_back('}');
        return *this;
    }
    Writer& begin_arr() {
        comma();
        out.push_back('[');
        return *this;
    }
    Writer& end_arr() {
        out.push_back(']');
        return *this;
    }
    // value helpers that manage commas inside arrays
    Writer& v(long long x) {
        comma();
        return num(x);
    }
    Writer& vd(double x) {
        comma();
        return dbl(x);
    }
    Writer& vs(const std::string& x) {
        comma();
        return str(x);
    }
    template <class T>
    Writer& ints(const std::vector<T>& xs) {
        begin_arr();
        for (const T& x : xs) v(static_cast<long long>(x));
        return end_arr();
    }

  private:
    void comma() {
        if (out.empty()) return;
        const char last = out.back();
        if (last != '[' && last != '{' && last != ':') out.push_back(',');
    }
};

}  // namespace json
}  // namespace pipetune
