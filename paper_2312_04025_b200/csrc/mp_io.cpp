// mp_io.cpp — native ingestion of schema-1 graph documents.
//
// Replaces the parse + object-construction half of fileio.load_graph
// (pkg/src/opplace/fileio.py:58-70, document layout :39-55) for C5-scale graphs:
// a single-pass streaming JSON reader writes the nodes and edges straight into
// flat arrays (ids, memory, tags, interned op types and type sequences, members,
// per-device compute times, edge list in file order) and runs the validations
// of OpNode / FlowEdge / CompGraph (graph.py:31-109).  Any document it cannot
// take on the fast path (a validation failure, a non-integer where the schema
// has integers, an unknown field type) is reported as MP_ERR_INVALID and the
// Python loader re-reads it, raising the reference's own exception.
//
// Numbers: integers as int64 (overflow -> MP_ERR_INVALID), reals with strtod
// (correctly rounded, as Python's float()); strings decode every JSON escape
// including \uXXXX surrogate pairs to UTF-8.

#include <cerrno>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/moirai_b200.h"

struct mp_graph_doc {
    std::vector<int64_t> id, mem, members, ct_dev, esrc, edst, epay;
    std::vector<int32_t> op_type, seq_beg, seq, mem_beg, ct_beg;
    std::vector<int8_t> tag;
    std::vector<double> ct_val;
    std::vector<int64_t> str_beg;
    std::string str;
};

namespace {

struct Fail {
    std::string msg;
};

struct Reader {
    const char *p, *e;
    std::unordered_map<std::string, int32_t> intern;
    mp_graph_doc *doc;

    [[noreturn]] void fail(const char *fmt, ...) {
        char buf[200];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        throw Fail{buf};
    }
    void ws() {
        while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    bool peek(char c) {
        ws();
        return p < e && *p == c;
    }
    void expect(char c) {
        ws();
        if (p >= e || *p != c) fail("expected '%c'", c);
        ++p;
    }
    static void utf8(std::string &out, unsigned cp) {
        if (cp < 0x80) {
            out += static_cast<char>(cp);
        } else if (cp < 0x800) {
            out += static_cast<char>(0xC0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += static_cast<char>(0xE0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        } else {
            out += static_cast<char>(0xF0 | (cp >> 18));
            out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
        }
    }
    unsigned hex4() {
        if (e - p < 4) fail("short \\u escape");
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            const char c = *p++;
            v <<= 4;
            if (c >= '0' && c <= '9') v |= c - '0';
            else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
            else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
            else fail("bad \\u escape");
        }
        return v;
    }
    std::string string() {
        expect('"');
        std::string out;
        while (true) {
            if (p >= e) fail("unterminated string");
            const char c = *p++;
            if (c == '"') break;
            if (c != '\\') {
                out += c;
                continue;
            }
            if (p >= e) fail("bad escape");
            const char x = *p++;
            switch (x) {
                case '"': out += '"'; break;
                case '\\': out += '\\'; break;
                case '/': out += '/'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'n': out += '\n'; break;
                case 'r': out += '\r'; break;
                case 't': out += '\t'; break;
                case 'u': {
                    unsigned cp = hex4();
                    if (cp >= 0xD800 && cp < 0xDC00 && e - p >= 6 && p[0] == '\\' && p[1] == 'u') {
                        p += 2;
                        const unsigned lo = hex4();
                        if (lo >= 0xDC00 && lo < 0xE000) cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        else fail("unpaired surrogate");
                    }
                    utf8(out, cp);
                    break;
                }
                default: fail("bad escape");
            }
        }
        return out;
    }
    // number: returns true if it is an integer literal (value in *iv), else a real in *dv
    bool number(long long *iv, double *dv) {
        ws();
        const char *s = p;
        if (p < e && (*p == '-' || *p == '+')) ++p;
        bool real = false;
        while (p < e && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' || *p == '-' || *p == '+')) {
            if (*p == '.' || *p == 'e' || *p == 'E') real = true;
            ++p;
        }
        if (p == s) fail("expected a number");
        std::string tok(s, p);
        if (!real) {
            errno = 0;
            char *end = nullptr;
            const long long v = strtoll(tok.c_str(), &end, 10);
            if (errno || *end) fail("integer out of range");
            *iv = v;
            *dv = static_cast<double>(v);
            return true;
        }
        char *end = nullptr;
        *dv = strtod(tok.c_str(), &end);
        if (*end) fail("bad number");
        return false;
    }
    long long integer() {
        long long v;
        double d;
        if (!number(&v, &d)) fail("expected an integer");
        return v;
    }
    double real() {  // float(x) of an int or a real
        long long v;
        double d;
        ws();
        if (p < e && *p == '"') fail("expected a number");
        // Python's float(int) and the int64 -> double conversion both round to nearest
        return number(&v, &d) ? static_cast<double>(v) : d;
    }
    void skip() {
        ws();
        if (p >= e) fail("unexpected end");
        if (*p == '"') {
            string();
        } else if (*p == '{') {
            ++p;
            if (peek('}')) {
                ++p;
                return;
            }
            do {
                string();
                expect(':');
                skip();
            } while (comma());
            expect('}');
        } else if (*p == '[') {
            ++p;
            if (peek(']')) {
                ++p;
                return;
            }
            do skip();
            while (comma());
            expect(']');
        } else if (!strncmp(p, "true", 4) && e - p >= 4) {
            p += 4;
        } else if (!strncmp(p, "false", 5) && e - p >= 5) {
            p += 5;
        } else if (!strncmp(p, "null", 4) && e - p >= 4) {
            p += 4;
        } else {
            long long v;
            double d;
            number(&v, &d);
        }
    }
    bool comma() {
        ws();
        if (p < e && *p == ',') {
            ++p;
            return true;
        }
        return false;
    }
    int32_t intern_str(const std::string &s) {
        auto it = intern.find(s);
        if (it != intern.end()) return it->second;
        const int32_t k = static_cast<int32_t>(doc->str_beg.size() - 1);
        doc->str += s;
        doc->str_beg.push_back(static_cast<int64_t>(doc->str.size()));
        intern.emplace(s, k);
        return k;
    }

    void node() {
        mp_graph_doc &d = *doc;
        bool have_id = false, have_type = false, have_mem = false, have_ct = false;
        long long id = 0, mem = 0;
        int32_t ty = -1;
        int8_t tag = 0;
        std::vector<int64_t> members;
        std::vector<int32_t> seq;
        std::vector<std::pair<int64_t, double>> ct;
        expect('{');
        if (!peek('}')) {
            do {
                const std::string key = string();
                expect(':');
                if (key == "id") {
                    id = integer();
                    have_id = true;
                } else if (key == "op_type") {
                    ty = intern_str(string());
                    have_type = true;
                } else if (key == "mem_bytes") {
                    mem = integer();
                    have_mem = true;
                } else if (key == "tag") {
                    const std::string t = string();
                    if (t == "plain") tag = 0;
                    else if (t == "fused") tag = 1;
                    else if (t == "bound") tag = 2;
                    else fail("unknown tag");
                } else if (key == "members") {
                    expect('[');
                    if (!peek(']')) {
                        do members.push_back(integer());
                        while (comma());
                    }
                    expect(']');
                } else if (key == "type_seq") {
                    expect('[');
                    if (!peek(']')) {
                        do seq.push_back(intern_str(string()));
                        while (comma());
                    }
                    expect(']');
                } else if (key == "compute_time") {
                    have_ct = true;
                    expect('{');
                    if (!peek('}')) {
                        do {
                            const std::string k = string();
                            char *end = nullptr;
                            errno = 0;
                            const long long dev = strtoll(k.c_str(), &end, 10);
                            if (k.empty() || *end || errno) fail("device key is not an integer");
                            expect(':');
                            ct.emplace_back(dev, real());
                        } while (comma());
                    }
                    expect('}');
                } else {
                    skip();
                }
            } while (comma());
        }
        expect('}');
        if (!have_id || !have_type || !have_mem || !have_ct) fail("node lacks a required field");
        // OpNode.__post_init__ (graph.py:31-61)
        if (members.empty()) members.push_back(id);
        if (seq.empty()) seq.push_back(ty);
        if (mem < 0) fail("negative mem_bytes");
        if (members.size() != seq.size()) fail("members / type_seq length");
        {
            std::unordered_set<int64_t> u(members.begin(), members.end());
            if (u.size() != members.size()) fail("duplicate member ids");
        }
        for (auto &kv : ct)
            if (kv.second < 0 || std::isnan(kv.second)) fail("negative compute time");
        d.id.push_back(id);
        d.mem.push_back(mem);
        d.op_type.push_back(ty);
        d.tag.push_back(tag);
        d.members.insert(d.members.end(), members.begin(), members.end());
        d.mem_beg.push_back(static_cast<int32_t>(d.members.size()));
        d.seq.insert(d.seq.end(), seq.begin(), seq.end());
        d.seq_beg.push_back(static_cast<int32_t>(d.seq.size()));
        for (auto &kv : ct) {
            d.ct_dev.push_back(kv.first);
            d.ct_val.push_back(kv.second);
        }
        d.ct_beg.push_back(static_cast<int32_t>(d.ct_dev.size()));
    }

    void edge() {
        bool hs = false, hd = false, hp = false;
        long long s = 0, t = 0, pl = 0;
        expect('{');
        if (!peek('}')) {
            do {
                const std::string key = string();
                expect(':');
                if (key == "src") {
                    s = integer();
                    hs = true;
                } else if (key == "dst") {
                    t = integer();
                    hd = true;
                } else if (key == "payload_bytes") {
                    pl = integer();
                    hp = true;
                } else {
                    skip();
                }
            } while (comma());
        }
        expect('}');
        if (!hs || !hd || !hp) fail("edge lacks a required field");
        if (s == t) fail("self edge");
        if (pl < 0) fail("negative payload");
        doc->esrc.push_back(s);
        doc->edst.push_back(t);
        doc->epay.push_back(pl);
    }

    void document() {
        bool schema_ok = false, kind_ok = false, have_nodes = false, have_edges = false;
        expect('{');
        if (!peek('}')) {
            do {
                const std::string key = string();
                expect(':');
                if (key == "schema") {
                    long long v;
                    double dv;
                    ws();
                    schema_ok = (p < e && *p != '"' && number(&v, &dv) && v == 1);
                    if (!schema_ok) fail("unsupported schema");
                } else if (key == "kind") {
                    kind_ok = string() == "graph";
                    if (!kind_ok) fail("not a graph document");
                } else if (key == "nodes") {
                    have_nodes = true;
                    expect('[');
                    if (!peek(']')) {
                        do node();
                        while (comma());
                    }
                    expect(']');
                } else if (key == "edges") {
                    have_edges = true;
                    expect('[');
                    if (!peek(']')) {
                        do edge();
                        while (comma());
                    }
                    expect(']');
                } else {
                    skip();
                }
            } while (comma());
        }
        expect('}');
        ws();
        if (p != e) fail("trailing data");
        if (!schema_ok || !kind_ok || !have_nodes || !have_edges) fail("incomplete graph document");
        // CompGraph.__init__ (graph.py:87-109): unique ids, existing endpoints, no parallel edges
        std::unordered_set<int64_t> ids;
        ids.reserve(doc->id.size() * 2);
        for (int64_t x : doc->id)
            if (!ids.insert(x).second) fail("duplicate node id");
        std::unordered_set<unsigned long long> pairs;
        pairs.reserve(doc->esrc.size() * 2);
        for (size_t k = 0; k < doc->esrc.size(); ++k) {
            if (!ids.count(doc->esrc[k]) || !ids.count(doc->edst[k])) fail("dangling edge");
            const unsigned long long key = (static_cast<unsigned long long>(doc->esrc[k]) * 0x9E3779B97F4A7C15ULL) ^
                                           static_cast<unsigned long long>(doc->edst[k]);
            if (!pairs.insert(key).second) {
                // hash collision or a real parallel edge: check exactly
                for (size_t j = 0; j < k; ++j)
                    if (doc->esrc[j] == doc->esrc[k] && doc->edst[j] == doc->edst[k]) fail("parallel edge");
            }
        }
    }
};

int set_err(mp_error *err, int code, const std::string &msg) {
    if (err) {
        err->code = code;
        err->a = 0;
        err->b = 0;
        snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
    }
    return code;
}

}  // namespace

extern "C" int32_t mp_graph_load_json(const char *path, mp_graph_doc **out, mp_graph_view *view, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!path || !out || !view) return set_err(err, MP_ERR_INVALID, "null argument");
    *out = nullptr;
    FILE *f = fopen(path, "rb");
    if (!f) return set_err(err, MP_ERR_INVALID, std::string("cannot open ") + path);
    std::string buf;
    fseek(f, 0, SEEK_END);
    const long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
    const size_t got = sz > 0 ? fread(&buf[0], 1, buf.size(), f) : 0;
    fclose(f);
    if (got != buf.size()) return set_err(err, MP_ERR_INVALID, "short read");
    auto *doc = new mp_graph_doc();
    doc->seq_beg.push_back(0);
    doc->mem_beg.push_back(0);
    doc->ct_beg.push_back(0);
    doc->str_beg.push_back(0);
    Reader r{buf.data(), buf.data() + buf.size(), {}, doc};
    try {
        r.document();
    } catch (const Fail &x) {
        delete doc;
        return set_err(err, MP_ERR_INVALID, x.msg);
    }
    *out = doc;
    view->n_nodes = static_cast<int64_t>(doc->id.size());
    view->n_edges = static_cast<int64_t>(doc->esrc.size());
    view->n_strings = static_cast<int64_t>(doc->str_beg.size() - 1);
    view->id = doc->id.data();
    view->mem = doc->mem.data();
    view->tag = doc->tag.data();
    view->op_type = doc->op_type.data();
    view->seq_beg = doc->seq_beg.data();
    view->seq = doc->seq.data();
    view->mem_beg = doc->mem_beg.data();
    view->members = doc->members.data();
    view->ct_beg = doc->ct_beg.data();
    view->ct_dev = doc->ct_dev.data();
    view->ct_val = doc->ct_val.data();
    view->esrc = doc->esrc.data();
    view->edst = doc->edst.data();
    view->epay = doc->epay.data();
    view->str_beg = doc->str_beg.data();
    view->str = doc->str.data();
    return MP_OK;
}

extern "C" void mp_graph_doc_free(mp_graph_doc *doc) { delete doc; }
