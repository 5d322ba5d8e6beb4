#include "json_in.h"

#include <cctype>
#include <cstdlib>

namespace pipetune {
namespace json {

namespace {

struct Parser {
    const std::string& t;
    size_t p = 0;

    [[noreturn]] void fail(const std::string& why) const {
        // line-precise message
        int line = 1;
        for (size_t i = 0; i < p && i < t.size(); ++i) line += t[i] == '\n';
        throw ConfigError("JSON line " + std::to_string(line) + ": " + why);
    }
    void ws() {
        while (p < t.size() && std::isspace(static_cast<unsigned char>(t[p]))) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < t.size() && t[p] == c) {
            ++p;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    Value value() {
        ws();
        if (p >= t.size()) fail("unexpected end of input");
        const char c = t[p];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') {
            Value v;
            v.kind = Value::String;
            v.s = string();
            return v;
        }
        if (t.compare(p, 4, "true") == 0) {
            p += 4;
            Value v;
            v.kind = Value::Bool;
            v.b = true;
            return v;
        }
        if (t.compare(p, 5, "false") == 0) {
            p += 5;
            Value v;
            v.kind = Value::Bool;
            return v;
        }
        if (t.compare(p, 4, "null") == 0) {
            p += 4;
            return Value{};
        }
        return number();
    }
    std::string string() {
        expect('"');
        std::string out;
        while (p < t.size() && t[p] != '"') {
            char c = t[p++];
            if (c == '\\') {
                if (p >= t.size()) fail("bad escape");
                const char e = t[p++];
                switch (e) {
                    case 'n': out.push_back('\n'); break;
                    case 't': out.push_back('\t'); break;
                    case 'r': out.push_back('\r'); break;
                    case 'b': out.push_back('\b'); break;
                    case 'f': out.push_back('\f'); break;
                    case 'u': fail("\\u escapes are not supported");
                    default: out.push_back(e); break;
                }
            } else {
                out.push_back(c);
            }
        }
        if (p >= t.size()) fail("unterminated string");
        ++p;
        return out;
    }
    Value number() {
        const size_t s = p;
        if (p < t.size() && (t[p] == '-' || t[p] == '+')) ++p;
        bool frac = false;
        while (p < t.size() && (std::isdigit(static_cast<unsigned char>(t[p])) || t[p] == '.' || t[p] == 'e' ||
                                t[p] == 'E' || t[p] == '-' || t[p] == '+')) {
            if (t[p] == '.' || t[p] == 'e' || t[p] == 'E') frac = true;
            ++p;
        }
        if (s == p) fail("unexpected character");
        const std::string tok = t.substr(s, p - s);
        Value v;
        v.kind = Value::Number;
        char* end = nullptr;
        v.num = std::strtod(tok.c_str(), &end);
        if (end == nullptr || *end != '\0') fail("bad number '" + tok + "'");
        if (!frac) {
            v.is_int = true;
            v.i = std::strtoll(tok.c_str(), nullptr, 10);
        } else if (v.num == static_cast<double>(static_cast<long long>(v.num)) && v.num < 9.2e18 && v.num > -9.2e18) {
            v.is_int = true;  // e.g. 1e18 written in exponent form
            v.i = static_cast<long long>(v.num);
        }
        return v;
    }
    Value array() {
        expect('[');
        Value v;
        v.kind = Value::Array;
        if (eat(']')) return v;
        do v.arr.push_back(value());
        while (eat(','));
        expect(']');
        return v;
    }
    Value object() {
        expect('{');
        Value v;
        v.kind = Value::Object;
        if (eat('}')) return v;
        do {
            ws();
            std::string k = string();
            for (const auto& kv : v.obj)
                if (kv.first == k) fail("duplicate key '" + k + "'");
            expect(':');
            v.obj.emplace_back(std::move(k), value());
        } while (eat(','));
        expect('}');
        return v;
    }
};

}  // namespace

Value parse(const std::string& text) {
    Parser ps{text};
    Value v = ps.value();
    ps.ws();
    if (ps.p != text.size()) ps.fail("trailing characters");
    return v;
}

void require_keys(const Value& v, const char* where, std::initializer_list<const char*> allowed) {
    if (v.kind != Value::Object) throw ConfigError(std::string(where) + ": expected an object");
    for (const auto& kv : v.obj) {
        bool ok = false;
        for (const char* a : allowed) ok = ok || kv.first == a;
        if (!ok) throw ConfigError(std::string(where) + ": unknown key '" + kv.first + "'");
    }
}

}  // namespace json
}  // namespace pipetune
