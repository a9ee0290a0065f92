// json_min.h — minimal JSON reader for geometry files (objects, arrays, strings, numbers, literals).
#pragma once

#include <stdlib.h>
#include <string.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

namespace mig {
namespace json {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Value> arr;
    std::map<std::string, Value> obj;

    const Value* get(const std::string& k) const {
        if (kind != Object) return nullptr;
        auto it = obj.find(k);
        return it == obj.end() ? nullptr : &it->second;
    }
};

class Parser {
  public:
    explicit Parser(const std::string& s) : s_(s) {}

    // Returns false and sets err (with byte offset) on malformed input.
    bool parse(Value* out, std::string* err) {
        pos_ = 0;
        ws();
        if (!value(out, 0)) {
            *err = err_.empty() ? "syntax error" : err_;
            *err += " at byte " + std::to_string(pos_);
            return false;
        }
        ws();
        if (pos_ != s_.size()) {
            *err = "trailing characters at byte " + std::to_string(pos_);
            return false;
        }
        return true;
    }

  private:
    const std::string& s_;
    size_t pos_ = 0;
    std::string err_;

    void ws() {
        while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\n' || s_[pos_] == '\r' || s_[pos_] == '\t'))
            ++pos_;
    }
    bool lit(const char* w) {
        size_t n = strlen(w);
        if (s_.compare(pos_, n, w) != 0) return false;
        pos_ += n;
        return true;
    }
    bool value(Value* v, int depth) {
        if (depth > 64) {
            err_ = "nesting too deep";
            return false;
        }
        if (pos_ >= s_.size()) {
            err_ = "unexpected end";
            return false;
        }
        char c = s_[pos_];
        if (c == '{') return object(v, depth);
        if (c == '[') return array(v, depth);
        if (c == '"') {
            v->kind = Value::String;
            return string(&v->str);
        }
        if (lit("true")) {
            v->kind = Value::Bool;
            v->b = true;
            return true;
        }
        if (lit("false")) {
            v->kind = Value::Bool;
            return true;
        }
        if (lit("null")) return true;
        return number(v);
    }
    bool string(std::string* out) {
        ++pos_;  // opening quote
        while (pos_ < s_.size() && s_[pos_] != '"') {
            char c = s_[pos_++];
            if (c == '\\') {
                if (pos_ >= s_.size()) break;
                char e = s_[pos_++];
                switch (e) {
                    case 'n': out->push_back('\n'); break;
                    case 't': out->push_back('\t'); break;
                    case 'u': pos_ += 4; out->push_back('?'); break;
                    default: out->push_back(e);
                }
            } else {
                out->push_back(c);
            }
        }
        if (pos_ >= s_.size()) {
            err_ = "unterminated string";
            return false;
        }
        ++pos_;
        return true;
    }
    bool number(Value* v) {
        const char* b = s_.c_str() + pos_;
        char* e = nullptr;
        double d = strtod(b, &e);
        if (e == b) {
            err_ = "unexpected character";
            return false;
        }
        pos_ += (size_t)(e - b);
        v->kind = Value::Number;
        v->num = d;
        return true;
    }
    bool array(Value* v, int depth) {
        v->kind = Value::Array;
        ++pos_;
        ws();
        if (pos_ < s_.size() && s_[pos_] == ']') {
            ++pos_;
            return true;
        }
        for (;;) {
            Value x;
            ws();
            if (!value(&x, depth + 1)) return false;
            v->arr.push_back(std::move(x));
            ws();
            if (pos_ < s_.size() && s_[pos_] == ',') {
                ++pos_;
                continue;
            }
            if (pos_ < s_.size() && s_[pos_] == ']') {
                ++pos_;
                return true;
            }
            err_ = "expected ',' or ']'";
            return false;
        }
    }
    bool object(Value* v, int depth) {
        v->kind = Value::Object;
        ++pos_;
        ws();
        if (pos_ < s_.size() && s_[pos_] == '}') {
            ++pos_;
            return true;
        }
        for (;;) {
            ws();
            if (pos_ >= s_.size() || s_[pos_] != '"') {
                err_ = "expected key";
                return false;
            }
            std::string k;
            if (!string(&k)) return false;
            ws();
            if (pos_ >= s_.size() || s_[pos_] != ':') {
                err_ = "expected ':'";
                return false;
            }
            ++pos_;
            ws();
            Value x;
            if (!value(&x, depth + 1)) return false;
            v->obj[k] = std::move(x);
            ws();
            if (pos_ < s_.size() && s_[pos_] == ',') {
                ++pos_;
                continue;
            }
            if (pos_ < s_.size() && s_[pos_] == '}') {
                ++pos_;
                return true;
            }
            err_ = "expected ',' or '}'";
            return false;
        }
    }
};

}  // namespace json
}  // namespace mig
