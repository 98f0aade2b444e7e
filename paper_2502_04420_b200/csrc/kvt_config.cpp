// kvt_config.cpp — a1: loading the searched layer-wise configuration (host only).
//
// The configuration is the per-layer precision pair P = (P_k^l, P_v^l) of the MOO problem
// (Eq. 4), searched offline and "directly loaded without any additional overhead"
// (P:113).  JSON schema after S:471 (see include/kvt.h).  f_m = sum (b_k + b_v) / (2L) is
// recomputed from the layer list.
#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "kvt_internal.h"

struct kvt_config {
    std::string model_name;
    double label_bits = 0.0;
    double fm = 0.0;
    std::vector<kvt_layer_spec> layers;
};

namespace {

// ------------------------------------------------------------------------------------------------
// Minimal JSON reader (objects, arrays, strings, numbers, true/false/null) with line:col errors.
// ------------------------------------------------------------------------------------------------
struct JValue {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    bool is_int = false;
    std::string str;
    std::vector<JValue> arr;
    std::vector<std::pair<std::string, JValue>> obj;
    int line = 1, col = 1;
    const JValue* get(const char* key) const {
        for (auto& kv : obj) if (kv.first == key) return &kv.second;
        return nullptr;
    }
};

struct Parser {
    const std::string& s;
    size_t i = 0;
    int line = 1, col = 1;
    std::string err;
    explicit Parser(const std::string& src) : s(src) {}

    bool error(const char* what) {
        if (err.empty()) {
            char buf[256];
            std::snprintf(buf, sizeof buf, "JSON parse error at line %d, column %d: %s", line, col, what);
            err = buf;
        }
        return false;
    }
    void adv() {
        if (s[i] == '\n') { ++line; col = 1; } else { ++col; }
        ++i;
    }
    void ws() { while (i < s.size() && std::isspace((unsigned char)s[i])) adv(); }
    bool lit(const char* w) {
        size_t n = std::strlen(w);
        if (s.compare(i, n, w) != 0) return false;
        for (size_t k = 0; k < n; ++k) adv();
        return true;
    }
    bool value(JValue& v, int depth = 0) {
        if (depth > 64) return error("nesting too deep");
        ws();
        v.line = line; v.col = col;
        if (i >= s.size()) return error("unexpected end of input");
        char c = s[i];
        if (c == '{') {
            v.kind = JValue::Obj; adv(); ws();
            if (i < s.size() && s[i] == '}') { adv(); return true; }
            for (;;) {
                ws();
                JValue key;
                if (i >= s.size() || s[i] != '"') return error("expected object key string");
                if (!string(key.str)) return false;
                ws();
                if (i >= s.size() || s[i] != ':') return error("expected ':'");
                adv();
                JValue val;
                if (!value(val, depth + 1)) return false;
                v.obj.emplace_back(key.str, std::move(val));
                ws();
                if (i < s.size() && s[i] == ',') { adv(); continue; }
                if (i < s.size() && s[i] == '}') { adv(); return true; }
                return error("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JValue::Arr; adv(); ws();
            if (i < s.size() && s[i] == ']') { adv(); return true; }
            for (;;) {
                JValue el;
                if (!value(el, depth + 1)) return false;
                v.arr.push_back(std::move(el));
                ws();
                if (i < s.size() && s[i] == ',') { adv(); continue; }
                if (i < s.size() && s[i] == ']') { adv(); return true; }
                return error("expected ',' or ']'");
            }
        }
        if (c == '"') { v.kind = JValue::Str; return string(v.str); }
        if (lit("true")) { v.kind = JValue::Bool; v.b = true; return true; }
        if (lit("false")) { v.kind = JValue::Bool; v.b = false; return true; }
        if (lit("null")) { v.kind = JValue::Null; return true; }
        if (c == '-' || std::isdigit((unsigned char)c)) {
            size_t st = i;
            bool frac = false;
            if (s[i] == '-') adv();
            while (i < s.size() && (std::isdigit((unsigned char)s[i]) || s[i] == '.' || s[i] == 'e' ||
                                    s[i] == 'E' || s[i] == '+' || s[i] == '-')) {
                if (s[i] == '.' || s[i] == 'e' || s[i] == 'E') frac = true;
                adv();
            }
            std::string tok = s.substr(st, i - st);
            char* end = nullptr;
            v.num = std::strtod(tok.c_str(), &end);
            if (!end || *end != '\0') return error("malformed number");
            v.kind = JValue::Num;
            v.is_int = !frac;
            return true;
        }
        return error("unexpected character");
    }
    bool string(std::string& out) {
        adv();  // opening quote
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                adv();
                if (i >= s.size()) break;
                char e = s[i];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (i + 4 >= s.size()) return error("bad \\u escape");
                        unsigned cp = (unsigned)std::strtoul(s.substr(i + 1, 4).c_str(), nullptr, 16);
                        for (int k = 0; k < 4; ++k) adv();
                        if (cp < 0x80) out += (char)cp; else out += '?';
                        break;
                    }
                    default: return error("bad escape");
                }
                adv();
            } else {
                out += s[i];
                adv();
            }
        }
        if (i >= s.size()) return error("unterminated string");
        adv();
        return true;
    }
};

int32_t schema_err(const JValue* v, const char* what) {
    if (v) return kvt::fail(KVT_ERR_PARSE, "config schema error at line %d, column %d: %s", v->line, v->col, what);
    return kvt::fail(KVT_ERR_PARSE, "config schema error: %s", what);
}

bool get_int(const JValue* v, int64_t* out) {
    if (!v || v->kind != JValue::Num || !v->is_int) return false;
    *out = (int64_t)v->num;
    return true;
}

}  // namespace

extern "C" int32_t kvt_config_load(const char* path_or_json, kvt_config** out) {
    kvt::clear_error();
    if (!path_or_json || !out) return kvt::fail(KVT_ERR_INVALID_ARG, "kvt_config_load: null argument");
    *out = nullptr;
    std::string text;
    const char* p = path_or_json;
    while (*p && std::isspace((unsigned char)*p)) ++p;
    if (*p == '{') {
        text = p;
    } else {
        std::ifstream f(path_or_json, std::ios::binary);
        if (!f) return kvt::fail(KVT_ERR_IO, "kvt_config_load: cannot open '%s'", path_or_json);
        std::stringstream ss;
        ss << f.rdbuf();
        text = ss.str();
    }
    JValue root;
    Parser ps(text);
    if (!ps.value(root)) return kvt::fail(KVT_ERR_PARSE, "%s", ps.err.c_str());
    ps.ws();
    if (ps.i != text.size()) { ps.error("trailing characters after the document"); return kvt::fail(KVT_ERR_PARSE, "%s", ps.err.c_str()); }
    if (root.kind != JValue::Obj) return schema_err(&root, "top level must be an object");

    auto cfg = std::make_unique<kvt_config>();
    const JValue* mn = root.get("model_name");
    if (mn) {
        if (mn->kind != JValue::Str) return schema_err(mn, "\"model_name\" must be a string");
        cfg->model_name = mn->str;
    }
    const JValue* qm = root.get("quant_method");
    if (!qm || qm->kind != JValue::Str) return schema_err(qm ? qm : &root, "\"quant_method\" (string) is required");
    int mode;
    if (qm->str == "kivi" || qm->str == "KIVI") mode = KVT_MODE_KIVI;
    else if (qm->str == "per-token-asym") mode = KVT_MODE_PER_TOKEN_ASYM;
    else if (qm->str == "per-channel-asym")
        return kvt::fail(KVT_ERR_UNSUPPORTED, "quant_method \"per-channel-asym\" needs whole-sequence statistics and "
                                              "cannot be stored write-once (DESIGN.md §7)");
    else return schema_err(qm, "\"quant_method\" must be \"kivi\", \"per-token-asym\" or \"per-channel-asym\"");

    int64_t group = 32, residual = (mode == KVT_MODE_KIVI) ? 32 : 0;   // P:707 (KIVI); A5/A6
    if (const JValue* g = root.get("group_size")) {
        if (!get_int(g, &group) || group <= 0) return schema_err(g, "\"group_size\" must be a positive integer");
    }
    if (const JValue* r = root.get("residual_length")) {
        if (!get_int(r, &residual) || residual < 0) return schema_err(r, "\"residual_length\" must be a non-negative integer");
    }
    if (const JValue* eb = root.get("equivalent_bits")) {
        if (eb->kind != JValue::Num) return schema_err(eb, "\"equivalent_bits\" must be a number");
        cfg->label_bits = eb->num;
    }
    const JValue* layers = root.get("layers");
    if (!layers || layers->kind != JValue::Arr || layers->arr.empty())
        return schema_err(layers ? layers : &root, "\"layers\" must be a non-empty array");
    size_t L = layers->arr.size();
    std::vector<int> seen(L, 0);
    cfg->layers.assign(L, kvt_layer_spec{});
    double bits_sum = 0.0;
    for (const JValue& e : layers->arr) {
        if (e.kind != JValue::Obj) return schema_err(&e, "each layer entry must be an object");
        int64_t li, kb, vb;
        if (!get_int(e.get("layer"), &li)) return schema_err(&e, "layer entry needs integer \"layer\"");
        if (!get_int(e.get("key_bits"), &kb)) return schema_err(&e, "layer entry needs integer \"key_bits\"");
        if (!get_int(e.get("value_bits"), &vb)) return schema_err(&e, "layer entry needs integer \"value_bits\"");
        if (li < 0 || (size_t)li >= L) return schema_err(&e, "\"layer\" out of range 0..L-1");
        if (seen[li]++) return schema_err(&e, "duplicate \"layer\" index");
        auto okb = [](int64_t b) { return b == 2 || b == 4 || b == 8 || b == 16; };
        if (!okb(kb) || !okb(vb)) return schema_err(&e, "bits must be one of 2, 4, 8, 16 (P:316; 16 = bf16)");
        kvt_layer_spec& s = cfg->layers[li];
        s.mode = mode; s.key_bits = (int32_t)kb; s.value_bits = (int32_t)vb;
        s.group = (int32_t)group; s.residual = (int32_t)residual;
        bits_sum += (double)(kb + vb);
    }
    if (mode == KVT_MODE_KIVI && residual % group != 0)
        return schema_err(&root, "kivi needs residual_length % group_size == 0 (blocks of G are flushed)");
    cfg->fm = bits_sum / (2.0 * (double)L);                              // f_m, Eq. 4
    *out = cfg.release();
    return KVT_OK;
}

extern "C" int32_t kvt_config_num_layers(const kvt_config* cfg) {
    return cfg ? (int32_t)cfg->layers.size() : -1;
}

extern "C" int32_t kvt_config_layer(const kvt_config* cfg, int32_t layer, kvt_layer_spec* out) {
    kvt::clear_error();
    if (!cfg || !out) return kvt::fail(KVT_ERR_INVALID_ARG, "kvt_config_layer: null argument");
    if (layer < 0 || (size_t)layer >= cfg->layers.size())
        return kvt::fail(KVT_ERR_INVALID_ARG, "kvt_config_layer: layer %d out of range", layer);
    *out = cfg->layers[layer];
    return KVT_OK;
}

extern "C" double kvt_config_equivalent_bits(const kvt_config* cfg) { return cfg ? cfg->fm : -1.0; }
extern "C" double kvt_config_label_bits(const kvt_config* cfg) { return cfg ? cfg->label_bits : -1.0; }
extern "C" const char* kvt_config_model_name(const kvt_config* cfg) { return cfg ? cfg->model_name.c_str() : ""; }
extern "C" void kvt_config_free(kvt_config* cfg) { delete cfg; }
