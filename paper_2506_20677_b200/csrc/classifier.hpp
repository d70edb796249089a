// classifier.hpp — NEXT-4 (host only): the strategy classifier of PAPER.md
// §III.H (Listing 5 loadModel / predictStrategy, lines 290-332; "combines ML
// predictions for n >= 1000 with static thresholds", Table IV) as portable
// tree-ensemble inference.  The format is SPEC.md's "ahs-model/1" JSON:
//   {"version":"ahs-model/1", "classes":[4 names], "feature_names":["n","k","H"],
//    "base_scores":[4 reals], "trees":[{"nodes":[node, ...]}, ...]}
//   node = {"feature":0..2, "threshold":real, "left":i, "right":i} | {"leaf":[4 reals]}
// Unknown fields are rejected; every tree is validated eagerly (children in
// range, no node reached twice from the root: a tree, acyclic).
// predict: score_c = base_c + sum over trees of the reached leaf's score_c,
// going left iff feature value < threshold; strategy = argmax, ties to the
// earlier class in `classes`.  The trained model is not part of this work
// (SURVEY §8(f)); tests use an FSM-consistent fixture (tests/golden).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace ahs {
namespace model {

// ------------------------------------------------------------------ JSON
struct JVal {
    enum Kind { NUL, BOOL, NUM, STR, ARR, OBJ } kind = NUL;
    bool b = false;
    double num = 0.0;
    bool integral = false;  // the literal had no fraction / exponent
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;
    const JVal *get(const char *key) const
    {
        for (const auto &kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
};

class Parser {
  public:
    Parser(const char *s, size_t n) : p_(s), end_(s + n) {}
    bool parse(JVal &out, std::string &err)
    {
        ws();
        if (!value(out, 0)) {
            err = err_.empty() ? "parse error" : err_;
            return false;
        }
        ws();
        if (p_ != end_) {
            err = "trailing characters after the JSON value";
            return false;
        }
        return true;
    }

  private:
    const char *p_, *end_;
    std::string err_;
    bool fail(const char *m)
    {
        if (err_.empty()) err_ = m;
        return false;
    }
    void ws()
    {
        while (p_ < end_ && (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r')) p_++;
    }
    bool lit(const char *w)
    {
        const size_t n = std::strlen(w);
        if ((size_t)(end_ - p_) < n || std::strncmp(p_, w, n) != 0) return fail("invalid literal");
        p_ += n;
        return true;
    }
    bool value(JVal &v, int depth)
    {
        if (depth > 64) return fail("nesting too deep");
        if (p_ >= end_) return fail("unexpected end of input");
        switch (*p_) {
        case '{': return object(v, depth);
        case '[': return array(v, depth);
        case '"': v.kind = JVal::STR; return string(v.str);
        case 't': v.kind = JVal::BOOL; v.b = true; return lit("true");
        case 'f': v.kind = JVal::BOOL; v.b = false; return lit("false");
        case 'n': v.kind = JVal::NUL; return lit("null");
        default: return number(v);
        }
    }
    bool object(JVal &v, int depth)
    {
        v.kind = JVal::OBJ;
        p_++;  // {
        ws();
        if (p_ < end_ && *p_ == '}') {
            p_++;
            return true;
        }
        for (;;) {
            ws();
            std::string key;
            if (p_ >= end_ || *p_ != '"' || !string(key)) return fail("expected a string key");
            for (const auto &kv : v.obj)
                if (kv.first == key) return fail("duplicate key");
            ws();
            if (p_ >= end_ || *p_ != ':') return fail("expected ':'");
            p_++;
            ws();
            JVal x;
            if (!value(x, depth + 1)) return false;
            v.obj.emplace_back(std::move(key), std::move(x));
            ws();
            if (p_ < end_ && *p_ == ',') {
                p_++;
                continue;
            }
            if (p_ < end_ && *p_ == '}') {
                p_++;
                return true;
            }
            return fail("expected ',' or '}'");
        }
    }
    bool array(JVal &v, int depth)
    {
        v.kind = JVal::ARR;
        p_++;  // [
        ws();
        if (p_ < end_ && *p_ == ']') {
            p_++;
            return true;
        }
        for (;;) {
            ws();
            JVal x;
            if (!value(x, depth + 1)) return false;
            v.arr.push_back(std::move(x));
            ws();
            if (p_ < end_ && *p_ == ',') {
                p_++;
                continue;
            }
            if (p_ < end_ && *p_ == ']') {
                p_++;
                return true;
            }
            return fail("expected ',' or ']'");
        }
    }
    bool string(std::string &s)
    {
        p_++;  // "
        while (p_ < end_ && *p_ != '"') {
            char c = *p_++;
            if ((unsigned char)c < 0x20) return fail("control character in string");
            if (c == '\\') {
                if (p_ >= end_) return fail("bad escape");
                const char e = *p_++;
                switch (e) {
                case '"': s += '"'; break;
                case '\\': s += '\\'; break;
                case '/': s += '/'; break;
                case 'b': s += '\b'; break;
                case 'f': s += '\f'; break;
                case 'n': s += '\n'; break;
                case 'r': s += '\r'; break;
                case 't': s += '\t'; break;
                case 'u': {
                    if (end_ - p_ < 4) return fail("bad \\u escape");
                    unsigned cp = 0;
                    for (int i = 0; i < 4; i++) {
                        const char h = *p_++;
                        cp = cp * 16 + (unsigned)(h >= '0' && h <= '9' ? h - '0'
                                                  : h >= 'a' && h <= 'f' ? h - 'a' + 10
                                                  : h >= 'A' && h <= 'F' ? h - 'A' + 10
                                                                         : 99);
                        if (cp > 0xffff) return fail("bad \\u escape");
                    }
                    if (cp >= 0x80) return fail("non-ASCII \\u escape not supported");
                    s += (char)cp;
                    break;
                }
                default: return fail("bad escape");
                }
            } else {
                s += c;
            }
        }
        if (p_ >= end_) return fail("unterminated string");
        p_++;  // "
        return true;
    }
    bool number(JVal &v)
    {
        const char *q = p_;
        if (q < end_ && *q == '-') q++;
        if (q >= end_ || !(*q >= '0' && *q <= '9')) return fail("invalid value");
        if (*q == '0') q++;
        else
            while (q < end_ && *q >= '0' && *q <= '9') q++;
        bool integral = true;
        if (q < end_ && *q == '.') {
            integral = false;
            q++;
            if (q >= end_ || !(*q >= '0' && *q <= '9')) return fail("invalid number");
            while (q < end_ && *q >= '0' && *q <= '9') q++;
        }
        if (q < end_ && (*q == 'e' || *q == 'E')) {
            integral = false;
            q++;
            if (q < end_ && (*q == '+' || *q == '-')) q++;
            if (q >= end_ || !(*q >= '0' && *q <= '9')) return fail("invalid number");
            while (q < end_ && *q >= '0' && *q <= '9') q++;
        }
        const std::string lit(p_, q);
        v.kind = JVal::NUM;
        v.num = std::strtod(lit.c_str(), nullptr);
        v.integral = integral;
        p_ = q;
        return true;
    }
};

// ----------------------------------------------------------------- model
enum Algo { INSERTION = 0, COUNTING = 1, RADIX = 2, QUICK = 3 };  // the paper's four (§III.A)

struct Node {
    int feature = -1;  // -1: leaf
    double threshold = 0.0;
    int left = -1, right = -1;
    double leaf[4] = {0, 0, 0, 0};
};

struct Model {
    int classes[4];  // class position -> Algo
    double base[4];
    std::vector<std::vector<Node>> trees;

    // scores in class order; returns the winning Algo
    int predict(double n, double k, double H, double scores[4]) const
    {
        const double x[3] = {n, k, H};
        for (int c = 0; c < 4; c++) scores[c] = base[c];
        for (const auto &t : trees) {
            int i = 0;
            while (t[i].feature >= 0) i = x[t[i].feature] < t[i].threshold ? t[i].left : t[i].right;
            for (int c = 0; c < 4; c++) scores[c] += t[i].leaf[c];
        }
        int best = 0;
        for (int c = 1; c < 4; c++)
            if (scores[c] > scores[best]) best = c;  // ties: the earlier class
        return classes[best];
    }
};

enum LoadStatus { LOAD_OK = 0, LOAD_PARSE = 1, LOAD_INVALID = 2, LOAD_VERSION = 3 };

inline bool only_keys(const JVal &o, std::initializer_list<const char *> keys)
{
    for (const auto &kv : o.obj) {
        bool ok = false;
        for (const char *k : keys) ok |= kv.first == k;
        if (!ok) return false;
    }
    return true;
}

inline bool finite_reals(const JVal *v, size_t n, double *out)
{
    if (!v || v->kind != JVal::ARR || v->arr.size() != n) return false;
    for (size_t i = 0; i < n; i++) {
        if (v->arr[i].kind != JVal::NUM || !std::isfinite(v->arr[i].num)) return false;
        out[i] = v->arr[i].num;
    }
    return true;
}

inline bool as_index(const JVal *v, long long lo, long long hi, int &out)
{
    if (!v || v->kind != JVal::NUM || !v->integral || v->num < (double)lo || v->num > (double)hi) return false;
    out = (int)v->num;
    return true;
}

inline LoadStatus load(const char *json, size_t len, Model &m, std::string &err)
{
    JVal root;
    Parser ps(json, len);
    if (!ps.parse(root, err)) return LOAD_PARSE;
    if (root.kind != JVal::OBJ) {
        err = "top level is not an object";
        return LOAD_INVALID;
    }
    if (!only_keys(root, {"version", "classes", "feature_names", "base_scores", "trees"})) {
        err = "unknown top-level field";
        return LOAD_INVALID;
    }
    const JVal *ver = root.get("version");
    if (!ver || ver->kind != JVal::STR) {
        err = "missing version";
        return LOAD_INVALID;
    }
    if (ver->str != "ahs-model/1") {
        err = "unsupported version '" + ver->str + "'";
        return LOAD_VERSION;
    }
    const JVal *cls = root.get("classes");
    if (!cls || cls->kind != JVal::ARR || cls->arr.size() != 4) {
        err = "classes must list 4 strategies";
        return LOAD_INVALID;
    }
    bool seen[4] = {false, false, false, false};
    for (int c = 0; c < 4; c++) {
        const JVal &e = cls->arr[c];
        int a = -1;
        if (e.kind == JVal::STR) {
            if (e.str == "insertion") a = INSERTION;
            else if (e.str == "counting") a = COUNTING;
            else if (e.str == "radix") a = RADIX;
            else if (e.str == "quick") a = QUICK;
        }
        if (a < 0 || seen[a]) {
            err = "classes must name insertion, counting, radix, quick once each";
            return LOAD_INVALID;
        }
        seen[a] = true;
        m.classes[c] = a;
    }
    const JVal *fn = root.get("feature_names");
    if (!fn || fn->kind != JVal::ARR || fn->arr.size() != 3 || fn->arr[0].str != "n" || fn->arr[1].str != "k" ||
        fn->arr[2].str != "H") {
        err = "feature_names must be [\"n\",\"k\",\"H\"]";
        return LOAD_INVALID;
    }
    if (!finite_reals(root.get("base_scores"), 4, m.base)) {
        err = "base_scores must be 4 finite reals";
        return LOAD_INVALID;
    }
    const JVal *trees = root.get("trees");
    if (!trees || trees->kind != JVal::ARR) {
        err = "trees must be an array";
        return LOAD_INVALID;
    }
    m.trees.clear();
    for (size_t t = 0; t < trees->arr.size(); t++) {
        const JVal &tv = trees->arr[t];
        const std::string where = "tree " + std::to_string(t);
        if (tv.kind != JVal::OBJ || !only_keys(tv, {"nodes"}) || !tv.get("nodes") ||
            tv.get("nodes")->kind != JVal::ARR || tv.get("nodes")->arr.empty()) {
            err = where + ": expected {\"nodes\": [...]} with at least one node";
            return LOAD_INVALID;
        }
        const auto &nodes = tv.get("nodes")->arr;
        const long long nn = (long long)nodes.size();
        std::vector<Node> out(nodes.size());
        for (size_t i = 0; i < nodes.size(); i++) {
            const JVal &nv = nodes[i];
            const std::string w = where + " node " + std::to_string(i);
            if (nv.kind != JVal::OBJ) {
                err = w + ": not an object";
                return LOAD_INVALID;
            }
            if (nv.get("leaf")) {
                if (!only_keys(nv, {"leaf"}) || !finite_reals(nv.get("leaf"), 4, out[i].leaf)) {
                    err = w + ": a leaf is {\"leaf\": [4 finite reals]}";
                    return LOAD_INVALID;
                }
                continue;
            }
            if (!only_keys(nv, {"feature", "threshold", "left", "right"}) ||
                !as_index(nv.get("feature"), 0, 2, out[i].feature)) {
                err = w + ": feature index must be 0, 1 or 2";
                return LOAD_INVALID;
            }
            const JVal *th = nv.get("threshold");
            if (!th || th->kind != JVal::NUM || !std::isfinite(th->num)) {
                err = w + ": threshold must be a finite real";
                return LOAD_INVALID;
            }
            out[i].threshold = th->num;
            if (!as_index(nv.get("left"), 0, nn - 1, out[i].left) ||
                !as_index(nv.get("right"), 0, nn - 1, out[i].right)) {
                err = w + ": child index out of range";
                return LOAD_INVALID;
            }
        }
        // a tree: walking from node 0 reaches no node twice (acyclic, no shared children)
        std::vector<char> seen_node(out.size(), 0);
        std::vector<int> stack{0};
        while (!stack.empty()) {
            const int i = stack.back();
            stack.pop_back();
            if (seen_node[i]) {
                err = where + ": node " + std::to_string(i) + " reached twice (not a tree)";
                return LOAD_INVALID;
            }
            seen_node[i] = 1;
            if (out[i].feature >= 0) {
                stack.push_back(out[i].left);
                stack.push_back(out[i].right);
            }
        }
        m.trees.push_back(std::move(out));
    }
    return LOAD_OK;
}

}  // namespace model
}  // namespace ahs
