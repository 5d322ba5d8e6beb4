// Small strict JSON reader for scenario configs.
// Integers keep exact int64 values; unknown-key rejection is done by callers.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "pipetune/errors.hpp"

namespace pipetune {
namespace json {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    bool is_int = false;
    long long i = 0;
    std::string s;
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;  // insertion order kept

    const Value* get(const std::string& k) const {
        for (const auto& kv : obj)
            if (kv.first == k) return &kv.second;
        return nullptr;
    }
    double as_double(const char* what) const {
        if (kind != Number) throw ConfigError(std::string("expected a number for ") + what);
        return num;
    }
    long long as_int(const char* what) const {
        if (kind != Number || !is_int) throw ConfigError(std::string("expected an integer for ") + what);
        return i;
    }
    const std::string& as_str(const char* what) const {
        if (kind != String) throw ConfigError(std::string("expected a string for ") + what);
        return s;
    }
    bool as_bool(const char* what) const {
        if (kind != Bool) throw ConfigError(std::string("expected a boolean for ") + what);
        return b;
    }
};

Value parse(const std::string& text);

// ConfigError listing the first key of `v` not in `allowed`.
void require_keys(const Value& v, const char* where, std::initializer_list<const char*> allowed);

}  // namespace json
}  // namespace pipetune
