// io.cpp — the reference's file formats on the host side of the boundary
// (SURVEY §8f rank 4): raw volumes with a JSON sidecar (io_raw.cpp:27-169)
// and the MDT2 binary checkpoint (checkpoint.cpp:24-145).  Files written here
// are byte-identical to the reference's writers (tests/test_io.py checks the
// goldens that oracle/gen_io_golden.sh makes with the reference's own code),
// and everything the reference writes loads here with the same checks and
// error classes (parse_error -> MDG_EPARSE, invalid_input -> MDG_EINVAL).
//
// JSON: a small reader for the two fixed schemas and writers that reproduce
// the reference's serializer output (nlohmann 3.11.3 as built in this image:
// sorted keys; dump(2) puts all-integer arrays on one line and other arrays
// one element per line; doubles as the shortest round-trip digits laid out
// with its decimal/exponent rules: 1.0, 0.0001, 1e-05, 1e+15).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mdg.h"

namespace mdg {
void set_error(mdg_status st, const std::string &msg);
}

namespace {

struct Fail {
    mdg_status st;
    std::string msg;
};
[[noreturn]] void parse_fail(const std::string &m) { throw Fail{MDG_EPARSE, m}; }
[[noreturn]] void input_fail(const std::string &m) { throw Fail{MDG_EINVAL, m}; }

template <class F>
mdg_status guarded(F &&f) {
    try {
        f();
        return MDG_OK;
    } catch (const Fail &e) {
        mdg::set_error(e.st, e.msg);
        return e.st;
    } catch (const std::exception &e) {
        mdg::set_error(MDG_EPARSE, e.what());
        return MDG_EPARSE;
    }
}

// ------------------------------------------------------------ JSON output
std::string fmt_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    std::string out;
    if (v < 0) {
        out = "-";
        v = -v;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
    const std::string sci(buf, r.ptr);  // d[.ddd]e±XX, shortest round trip
    const size_t e = sci.find('e');
    std::string digits = sci.substr(0, e);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = std::stoi(sci.substr(e + 1));
    const int k = (int)digits.size(), n = exp10 + 1;  // value = 0.digits * 10^n
    constexpr int kMin = -4, kMax = 15;
    if (k <= n && n <= kMax) {
        out += digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= kMax) {
        out += digits.substr(0, n) + "." + digits.substr(n);
    } else if (kMin < n && n <= 0) {
        out += "0." + std::string(-n, '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', std::abs(x));
        out += eb;
    }
    return out;
}

std::string sidecar_text(mdg_dims3 d, const float sp[3], const char *dtype, int channels) {
    std::string s = "{\n";
    if (channels != 1) s += "  \"channels\": " + std::to_string(channels) + ",\n";
    s += "  \"dims\": [" + std::to_string(d.h) + "," + std::to_string(d.w) + "," +
         std::to_string(d.l) + "],\n";
    s += std::string("  \"dtype\": \"") + dtype + "\",\n";
    s += "  \"order\": \"xyz-row-major\",\n";
    s += "  \"spacing\": [\n";
    for (int i = 0; i < 3; ++i)
        s += "    " + fmt_double((double)sp[i]) + (i < 2 ? ",\n" : "\n");
    s += "  ]\n}\n";
    return s;
}

std::string config_text(const mdg_model_config &c) {
    std::string s = "{\"base_channels\":" + std::to_string(c.base_channels);
    s += std::string(",\"diffeomorphic\":") + (c.diffeomorphic ? "true" : "false");
    s += ",\"head_dim\":" + std::to_string(c.head_dim);
    s += ",\"heads_per_level\":[";
    for (int i = 0; i < MDG_ENC_LEVELS; ++i)
        s += (i ? "," : "") + std::to_string(c.heads_per_level[i]);
    s += "],\"leaky_slope\":" + fmt_double((double)c.leaky_slope);
    s += ",\"neighborhood\":" + std::to_string(c.neighborhood);
    s += ",\"ss_steps\":" + std::to_string(c.ss_steps) + "}";
    return s;
}

// ------------------------------------------------------------- JSON input
struct JVal {
    enum Kind { Null, Bool, Int, Float, Str, Arr, Obj } kind = Null;
    bool b = false;
    int64_t i = 0;
    double f = 0.0;
    std::string s;
    std::vector<JVal> a;
    std::map<std::string, JVal> o;
    bool is_num() const { return kind == Int || kind == Float; }
    double num() const { return kind == Int ? (double)i : f; }
};

struct JParser {
    const char *p, *e;
    void ws() {
        while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    [[noreturn]] void bad(const char *what) { throw std::runtime_error(std::string("syntax error: ") + what); }
    JVal value() {
        ws();
        if (p >= e) bad("unexpected end of input");
        JVal v;
        if (*p == '{') {
            v.kind = JVal::Obj;
            ++p;
            ws();
            if (p < e && *p == '}') {
                ++p;
                return v;
            }
            for (;;) {
                ws();
                if (p >= e || *p != '"') bad("expected a key");
                std::string k = str();
                ws();
                if (p >= e || *p != ':') bad("expected ':'");
                ++p;
                v.o[k] = value();
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == '}') {
                    ++p;
                    return v;
                }
                bad("expected ',' or '}'");
            }
        }
        if (*p == '[') {
            v.kind = JVal::Arr;
            ++p;
            ws();
            if (p < e && *p == ']') {
                ++p;
                return v;
            }
            for (;;) {
                v.a.push_back(value());
                ws();
                if (p < e && *p == ',') {
                    ++p;
                    continue;
                }
                if (p < e && *p == ']') {
                    ++p;
                    return v;
                }
                bad("expected ',' or ']'");
            }
        }
        if (*p == '"') {
            v.kind = JVal::Str;
            v.s = str();
            return v;
        }
        if (e - p >= 4 && !std::strncmp(p, "true", 4)) {
            p += 4;
            v.kind = JVal::Bool;
            v.b = true;
            return v;
        }
        if (e - p >= 5 && !std::strncmp(p, "false", 5)) {
            p += 5;
            v.kind = JVal::Bool;
            return v;
        }
        if (e - p >= 4 && !std::strncmp(p, "null", 4)) {
            p += 4;
            return v;
        }
        const char *q = p;
        bool flt = false;
        if (q < e && (*q == '-' || *q == '+')) ++q;
        while (q < e && (std::isdigit((unsigned char)*q) || *q == '.' || *q == 'e' || *q == 'E' ||
                         *q == '-' || *q == '+')) {
            if (*q == '.' || *q == 'e' || *q == 'E') flt = true;
            ++q;
        }
        if (q == p) bad("unexpected character");
        const std::string t(p, q);
        p = q;
        if (flt) {
            v.kind = JVal::Float;
            v.f = std::stod(t);
        } else {
            v.kind = JVal::Int;
            v.i = std::stoll(t);
        }
        return v;
    }
    std::string str() {
        ++p;  // opening quote
        std::string s;
        while (p < e && *p != '"') {
            if (*p == '\\') {
                ++p;
                if (p >= e) bad("bad escape");
                const char c = *p;
                s += c == 'n' ? '\n' : c == 't' ? '\t' : c == 'r' ? '\r' : c;
            } else {
                s += *p;
            }
            ++p;
        }
        if (p >= e) bad("unterminated string");
        ++p;
        return s;
    }
};

JVal parse_json(const std::string &text) {
    JParser ps{text.data(), text.data() + text.size()};
    JVal v = ps.value();
    ps.ws();
    if (ps.p != ps.e) throw std::runtime_error("syntax error: trailing characters");
    return v;
}

const JVal &at(const JVal &o, const char *k) {
    auto it = o.o.find(k);
    if (o.kind != JVal::Obj || it == o.o.end())
        throw std::runtime_error(std::string("key '") + k + "' not found");
    return it->second;
}
int as_int(const JVal &v) {
    if (!v.is_num()) throw std::runtime_error("type must be number");
    return v.kind == JVal::Int ? (int)v.i : (int)v.f;
}
float as_float(const JVal &v) {
    if (!v.is_num()) throw std::runtime_error("type must be number");
    return (float)v.num();
}

// ------------------------------------------------------------------ files
std::vector<char> read_file(const std::string &path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) parse_fail("cannot open: " + path);
    const std::streamsize size = f.tellg();
    f.seekg(0);
    std::vector<char> buf((size_t)size);
    f.read(buf.data(), size);
    if (!f) parse_fail("short read: " + path);
    return buf;
}
void write_file(const std::string &path, const void *data, size_t bytes) {
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) parse_fail("cannot open for writing: " + path);
    f.write(static_cast<const char *>(data), (std::streamsize)bytes);
    if (!f) parse_fail("short write: " + path);
}

struct RawHeader {
    mdg_dims3 dims{0, 0, 0};
    float spacing[3] = {1.0f, 1.0f, 1.0f};
    std::string dtype;
    int channels = 1;
};

std::string data_path_for(const std::string &json_path) {
    const auto pos = json_path.rfind(".json");
    if (pos == std::string::npos || pos != json_path.size() - 5)
        input_fail("raw loader expects a .json sidecar path: " + json_path);
    return json_path.substr(0, pos) + ".raw";
}

RawHeader read_sidecar(const std::string &json_path) {
    const auto buf = read_file(json_path);
    JVal j;
    try {
        j = parse_json(std::string(buf.begin(), buf.end()));
    } catch (const std::exception &e) {
        parse_fail("invalid JSON sidecar " + json_path + ": " + e.what());
    }
    RawHeader h;
    try {
        const JVal &dims = at(j, "dims");
        if (dims.kind != JVal::Arr || dims.a.size() != 3)
            parse_fail("sidecar field 'dims' must have 3 entries");
        h.dims = mdg_dims3{as_int(dims.a[0]), as_int(dims.a[1]), as_int(dims.a[2])};
        const JVal &sp = at(j, "spacing");
        if (sp.kind != JVal::Arr || sp.a.size() < 3) throw std::runtime_error("spacing must be an array of 3");
        for (int i = 0; i < 3; ++i) h.spacing[i] = as_float(sp.a[i]);
        const JVal &dt = at(j, "dtype");
        if (dt.kind != JVal::Str) throw std::runtime_error("dtype must be a string");
        h.dtype = dt.s;
        const JVal &order = at(j, "order");
        if (order.kind != JVal::Str || order.s != "xyz-row-major")
            parse_fail("sidecar field 'order' must be xyz-row-major");
        auto it = j.o.find("channels");
        h.channels = it == j.o.end() ? 1 : as_int(it->second);
    } catch (const std::runtime_error &e) {
        parse_fail("sidecar " + json_path + " missing field: " + e.what());
    }
    if (h.dims.h < 1 || h.dims.w < 1 || h.dims.l < 1)
        parse_fail("sidecar field 'dims' must be positive");
    if (h.channels < 1) parse_fail("sidecar field 'channels' must be positive");
    return h;
}

std::vector<char> read_payload(const std::string &json_path, const RawHeader &h, size_t elem) {
    const std::string dpath = data_path_for(json_path);
    auto buf = read_file(dpath);
    const size_t expected = (size_t)h.dims.h * h.dims.w * h.dims.l * (size_t)h.channels * elem;
    if (buf.size() != expected)
        parse_fail("raw data length mismatch in " + dpath + ": expected " +
                   std::to_string(expected) + " bytes, got " + std::to_string(buf.size()));
    return buf;
}

void fill_header(const RawHeader &h, mdg_raw_header *out) {
    if (!out) return;
    out->dims = h.dims;
    for (int i = 0; i < 3; ++i) out->spacing[i] = h.spacing[i];
    out->dtype = h.dtype == "f32" ? MDG_RAW_F32 : h.dtype == "u16" ? MDG_RAW_U16 : -1;
    out->channels = h.channels;
}

mdg_status load_f32(const char *json_path, int channels, const char *what, mdg_raw_header *hdr,
                    float *out) {
    return guarded([&] {
        if (!json_path) input_fail("raw: null path");
        const std::string jp(json_path);
        const RawHeader h = read_sidecar(jp);
        if (h.dtype != "f32" || h.channels != channels)
            parse_fail(channels == 1 ? "expected a single-channel f32 raw volume: " + jp
                                     : "expected a 3-channel f32 raw field: " + jp);
        fill_header(h, hdr);
        if (!out) return;
        const auto buf = read_payload(jp, h, sizeof(float));
        std::memcpy(out, buf.data(), buf.size());
        const size_t n = buf.size() / sizeof(float);
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(out[i])) parse_fail(std::string("non-finite ") + what + " in " + jp);
    });
}

// ------------------------------------------------------------ checkpoints
struct TensorSpec {
    std::string name;
    std::vector<int> shape;
    int64_t n() const {
        int64_t v = 1;
        for (int d : shape) v *= d;
        return v;
    }
};

void validate_config(const mdg_model_config &c) {
    // ModelConfig::validate (engine.hpp:64-78) + EncoderConfig::validate
    if (c.base_channels < 1) input_fail("encoder: base_channels must be >= 1");
    for (int i = 0; i < MDG_ENC_LEVELS; ++i) {
        if (c.heads_per_level[i] < 1) input_fail("model: head counts must be >= 1");
        if (i > 0 && c.heads_per_level[i] > c.heads_per_level[i - 1])
            input_fail("model: head counts must be non-increasing coarse to fine");
    }
    if (c.head_dim < 1) input_fail("model: head_dim must be >= 1");
    if (c.neighborhood < 3 || c.neighborhood % 2 == 0)
        input_fail("model: neighborhood must be odd and >= 3");
    if (c.ss_steps < 1) input_fail("model: ss_steps must be >= 1");
}

// ModelParams::all_tensors (engine.hpp:121-133) names and shapes for a config
// (init_model engine.hpp:143-166, make_conv_block encoder.hpp:49-71,
// make_projection_params attention.hpp:330-343, make_reghead_params
// reghead.hpp:31-39)
std::vector<TensorSpec> layout_of(const mdg_model_config &c) {
    std::vector<TensorSpec> t;
    const int b = c.base_channels, L = MDG_ENC_LEVELS;
    for (int lv = 1; lv <= L; ++lv) {
        const int ic = lv == 1 ? 1 : b << (lv - 2), oc = b << (lv - 1);
        const std::string p = "enc.l" + std::to_string(lv);
        t.push_back({p + ".conv1.w", {oc, ic, 3, 3, 3}});
        t.push_back({p + ".conv1.b", {oc}});
        t.push_back({p + ".norm1.g", {oc}});
        t.push_back({p + ".norm1.b", {oc}});
        t.push_back({p + ".conv2.w", {oc, oc, 3, 3, 3}});
        t.push_back({p + ".conv2.b", {oc}});
        t.push_back({p + ".norm2.g", {oc}});
        t.push_back({p + ".norm2.b", {oc}});
    }
    const int win = c.neighborhood * c.neighborhood * c.neighborhood;
    for (int k = 0; k < L; ++k) {
        const int in_c = b << (L - k - 1), S = c.heads_per_level[k], K = S * c.head_dim;
        const std::string p = "lvl" + std::to_string(k);
        t.push_back({p + ".proj.w", {K, in_c}});
        t.push_back({p + ".proj.b", {K}});
        t.push_back({p + ".proj.ln_g", {K}});
        t.push_back({p + ".proj.ln_b", {K}});
        t.push_back({p + ".bias_b", {S, win}});
        t.push_back({p + ".reghead.w", {3, 3 * S, 3, 3, 3}});
        t.push_back({p + ".reghead.b", {3}});
    }
    return t;
}

mdg_model_config config_from_json(const std::string &text) {
    JVal j;
    try {
        j = parse_json(text);
    } catch (const std::exception &e) {
        parse_fail(std::string("invalid model config JSON: ") + e.what());
    }
    mdg_model_config c{};
    try {
        c.base_channels = as_int(at(j, "base_channels"));
        c.leaky_slope = as_float(at(j, "leaky_slope"));
        const JVal &h = at(j, "heads_per_level");
        if (h.kind != JVal::Arr) throw std::runtime_error("heads_per_level must be an array");
        if ((int)h.a.size() != MDG_ENC_LEVELS)
            input_fail("model: heads_per_level must have one entry per level");
        for (int i = 0; i < MDG_ENC_LEVELS; ++i) c.heads_per_level[i] = as_int(h.a[i]);
        c.head_dim = as_int(at(j, "head_dim"));
        c.neighborhood = as_int(at(j, "neighborhood"));
        const JVal &df = at(j, "diffeomorphic");
        if (df.kind != JVal::Bool) throw std::runtime_error("diffeomorphic must be a boolean");
        c.diffeomorphic = df.b ? 1 : 0;
        c.ss_steps = as_int(at(j, "ss_steps"));
    } catch (const std::runtime_error &e) {
        parse_fail(std::string("model config JSON missing field: ") + e.what());
    }
    validate_config(c);
    return c;
}

template <class T>
void put(std::string &s, T v) {
    s.append(reinterpret_cast<const char *>(&v), sizeof(T));
}
struct Reader {
    const std::vector<char> &b;
    size_t off = 0;
    template <class T>
    T get(const std::string &what) {
        if (off + sizeof(T) > b.size()) parse_fail("checkpoint truncated while reading " + what);
        T v;
        std::memcpy(&v, b.data() + off, sizeof(T));
        off += sizeof(T);
        return v;
    }
    std::string bytes(size_t n, const std::string &what) {
        if (off + n > b.size()) parse_fail("checkpoint truncated while reading " + what);
        std::string s(b.data() + off, n);
        off += n;
        return s;
    }
};

}  // namespace

extern "C" {

mdg_status mdg_model_config_small_preset(mdg_model_config *cfg) {
    if (!cfg) {
        mdg::set_error(MDG_EINVAL, "config: null pointer");
        return MDG_EINVAL;
    }
    // ModelConfig::small_preset (engine.hpp:38-44)
    *cfg = mdg_model_config{8, 0.2f, {8, 4, 2, 1, 1}, 6, 3, 0, 7};
    return MDG_OK;
}

int64_t mdg_config_param_count(const mdg_model_config *cfg, int *ntensors, int64_t *sizes) {
    if (!cfg) return -1;
    const auto t = layout_of(*cfg);
    if (ntensors) *ntensors = (int)t.size();
    int64_t tot = 0;
    for (size_t i = 0; i < t.size(); ++i) {
        if (sizes) sizes[i] = t[i].n();
        tot += t[i].n();
    }
    return tot;
}

mdg_status mdg_config_tensor_name(const mdg_model_config *cfg, int i, char *buf, int cap) {
    return guarded([&] {
        if (!cfg || !buf || cap < 1) input_fail("config: null pointer");
        const auto t = layout_of(*cfg);
        if (i < 0 || i >= (int)t.size()) input_fail("config: tensor index out of range");
        std::snprintf(buf, (size_t)cap, "%s", t[(size_t)i].name.c_str());
    });
}

mdg_status mdg_raw_load_volume(const char *json_path, mdg_raw_header *hdr, float *out) {
    return load_f32(json_path, 1, "voxel", hdr, out);
}

mdg_status mdg_raw_load_field(const char *json_path, mdg_raw_header *hdr, float *out) {
    return load_f32(json_path, 3, "displacement", hdr, out);
}

mdg_status mdg_raw_load_labels(const char *json_path, mdg_raw_header *hdr, int *out) {
    return guarded([&] {
        if (!json_path) input_fail("raw: null path");
        const std::string jp(json_path);
        const RawHeader h = read_sidecar(jp);
        if (h.dtype != "u16" || h.channels != 1)
            parse_fail("expected a single-channel u16 raw label volume: " + jp);
        fill_header(h, hdr);
        if (!out) return;
        const auto buf = read_payload(jp, h, sizeof(uint16_t));
        const size_t n = buf.size() / sizeof(uint16_t);
        for (size_t i = 0; i < n; ++i) {
            uint16_t v;
            std::memcpy(&v, buf.data() + 2 * i, 2);
            out[i] = v;
        }
    });
}

// load_nifti (nifti.cpp:36-105): single-file NIfTI-1, dim[0] = 3, datatype
// u8 / i16 / f32, scaled by scl_slope / scl_inter when scl_slope != 0
mdg_status mdg_nifti_load(const char *path, mdg_raw_header *hdr, float *out) {
    return guarded([&] {
        if (!path) input_fail("nifti: null path");
        const std::string ps(path);
        std::ifstream f(ps, std::ios::binary | std::ios::ate);
        if (!f) parse_fail("cannot open NIfTI file: " + ps);
        const std::streamsize size = f.tellg();
        if (size < 348) parse_fail("truncated NIfTI header in " + ps);
        f.close();
        const std::vector<char> buf = read_file(ps);
        auto rd = [&](size_t off, void *dst, size_t n) { std::memcpy(dst, buf.data() + off, n); };
        int32_t sizeof_hdr;
        rd(0, &sizeof_hdr, 4);
        if (sizeof_hdr != 348)
            parse_fail("bad NIfTI field sizeof_hdr (byte-swapped or invalid file)");
        if (!(buf[344] == 'n' && buf[345] == '+' && buf[346] == '1' && buf[347] == '\0'))
            parse_fail("bad NIfTI field magic: expected single-file magic n+1");
        int16_t dim[8];
        rd(40, dim, sizeof dim);
        if (dim[0] != 3)
            parse_fail("unsupported dimensionality: NIfTI field dim[0] = " + std::to_string(dim[0]));
        const mdg_dims3 d{dim[1], dim[2], dim[3]};
        if (d.h < 1 || d.w < 1 || d.l < 1) parse_fail("bad NIfTI field dim: non-positive extent");
        int16_t datatype, bitpix;
        rd(70, &datatype, 2);
        rd(72, &bitpix, 2);
        float pixdim[8], vox_offset, slope, inter;
        rd(76, pixdim, sizeof pixdim);
        rd(108, &vox_offset, 4);
        rd(112, &slope, 4);
        rd(116, &inter, 4);
        int elem = 0;
        switch (datatype) {
        case 2: elem = 1; break;
        case 4: elem = 2; break;
        case 16: elem = 4; break;
        default:
            parse_fail("unsupported NIfTI field datatype " + std::to_string(datatype) +
                       " (supported: 2, 4, 16)");
        }
        if (bitpix != elem * 8)
            parse_fail("bad NIfTI field bitpix " + std::to_string(bitpix) + " for datatype " +
                       std::to_string(datatype));
        const size_t offset = (size_t)vox_offset;
        if (vox_offset < 348.0f) parse_fail("bad NIfTI field vox_offset: " + std::to_string(vox_offset));
        const size_t nvox = (size_t)d.h * d.w * d.l;
        if (offset + nvox * (size_t)elem > buf.size())
            parse_fail("truncated NIfTI voxel data in " + ps);
        if (hdr) {
            hdr->dims = d;
            for (int i = 0; i < 3; ++i) hdr->spacing[i] = pixdim[i + 1] > 0.0f ? pixdim[i + 1] : 1.0f;
            hdr->dtype = MDG_RAW_F32;
            hdr->channels = 1;
        }
        if (!out) return;
        const bool scaled = slope != 0.0f;
        const char *base = buf.data() + offset;
        for (size_t i = 0; i < nvox; ++i) {
            float raw;
            if (datatype == 2) {
                raw = (float)(uint8_t)base[i];
            } else if (datatype == 4) {
                int16_t s16;
                std::memcpy(&s16, base + i * 2, 2);
                raw = (float)s16;
            } else {
                std::memcpy(&raw, base + i * 4, 4);
            }
            out[i] = scaled ? raw * slope + inter : raw;
            if (!std::isfinite(out[i])) parse_fail("non-finite voxel value in " + ps);
        }
    });
}

mdg_status mdg_raw_save_volume(const char *base, mdg_dims3 d, const float spacing[3],
                               const float *data) {
    return guarded([&] {
        if (!base || !spacing || !data) input_fail("raw: null pointer");
        const std::string b(base), text = sidecar_text(d, spacing, "f32", 1);
        write_file(b + ".json", text.data(), text.size());
        write_file(b + ".raw", data, (size_t)d.h * d.w * d.l * sizeof(float));
    });
}

mdg_status mdg_raw_save_field(const char *base, mdg_dims3 d, const float *data) {
    return guarded([&] {
        if (!base || !data) input_fail("raw: null pointer");
        const float one[3] = {1.0f, 1.0f, 1.0f};
        const std::string b(base), text = sidecar_text(d, one, "f32", 3);
        write_file(b + ".json", text.data(), text.size());
        write_file(b + ".raw", data, 3 * (size_t)d.h * d.w * d.l * sizeof(float));
    });
}

mdg_status mdg_raw_save_labels(const char *base, mdg_dims3 d, const float spacing[3],
                               const int *labels) {
    return guarded([&] {
        if (!base || !spacing || !labels) input_fail("raw: null pointer");
        const size_t n = (size_t)d.h * d.w * d.l;
        std::vector<uint16_t> packed(n);
        for (size_t i = 0; i < n; ++i) {
            if (labels[i] < 0 || labels[i] > 65535) input_fail("label value out of u16 range");
            packed[i] = (uint16_t)labels[i];
        }
        const std::string b(base), text = sidecar_text(d, spacing, "u16", 1);
        write_file(b + ".json", text.data(), text.size());
        write_file(b + ".raw", packed.data(), n * sizeof(uint16_t));
    });
}

mdg_status mdg_checkpoint_save(const char *path, const mdg_model_config *cfg,
                               const float *const *tensors) {
    return guarded([&] {
        if (!path || !cfg || !tensors) input_fail("checkpoint: null pointer");
        validate_config(*cfg);
        const auto specs = layout_of(*cfg);
        std::string s("MDT2", 4);
        put<uint32_t>(s, 1u);
        const std::string ct = config_text(*cfg);
        put<uint64_t>(s, ct.size());
        s += ct;
        put<uint32_t>(s, (uint32_t)specs.size());
        for (size_t i = 0; i < specs.size(); ++i) {
            if (!tensors[i]) input_fail("checkpoint: null tensor " + specs[i].name);
            put<uint32_t>(s, (uint32_t)specs[i].name.size());
            s += specs[i].name;
            put<uint32_t>(s, (uint32_t)specs[i].shape.size());
            for (int dim : specs[i].shape) put<uint32_t>(s, (uint32_t)dim);
            put<uint64_t>(s, (uint64_t)specs[i].n());
            s.append(reinterpret_cast<const char *>(tensors[i]), (size_t)specs[i].n() * sizeof(float));
        }
        write_file(path, s.data(), s.size());
    });
}

// config only (to size the tensor buffers) when tensors == NULL
mdg_status mdg_checkpoint_load(const char *path, mdg_model_config *cfg, float *const *tensors) {
    return guarded([&] {
        if (!path || !cfg) input_fail("checkpoint: null pointer");
        const std::string ps(path);
        std::vector<char> buf;
        {
            std::ifstream f(ps, std::ios::binary);
            if (!f) parse_fail("cannot open checkpoint: " + ps);
        }
        buf = read_file(ps);
        Reader r{buf};
        if (buf.size() < 4 || std::memcmp(buf.data(), "MDT2", 4) != 0)
            parse_fail("bad checkpoint magic in " + ps);
        r.off = 4;
        const auto version = r.get<uint32_t>("version");
        if (version != 1u) parse_fail("unsupported checkpoint version " + std::to_string(version));
        const auto clen = r.get<uint64_t>("config length");
        if (r.off + clen > buf.size()) parse_fail("checkpoint truncated while reading config");
        const mdg_model_config c = config_from_json(r.bytes((size_t)clen, "config"));
        *cfg = c;
        if (!tensors) return;
        const auto specs = layout_of(c);
        const auto count = r.get<uint32_t>("tensor count");
        if (count != specs.size())
            parse_fail("checkpoint tensor count " + std::to_string(count) +
                       " does not match model layout (" + std::to_string(specs.size()) + ")");
        for (size_t i = 0; i < specs.size(); ++i) {
            const auto nl = r.get<uint32_t>("tensor name length");
            if (r.off + nl > buf.size()) parse_fail("checkpoint truncated while reading tensor name");
            const std::string name = r.bytes(nl, "tensor name");
            if (name != specs[i].name)
                parse_fail("checkpoint tensor '" + name + "' does not match expected '" +
                           specs[i].name + "'");
            const auto nd = r.get<uint32_t>("tensor rank");
            std::vector<int> shape(nd);
            for (auto &dim : shape) dim = (int)r.get<uint32_t>("tensor dim");
            if (shape != specs[i].shape)
                parse_fail("checkpoint tensor '" + name + "' has unexpected shape");
            const auto n = r.get<uint64_t>("tensor size");
            if (n != (uint64_t)specs[i].n())
                parse_fail("checkpoint tensor '" + name + "' has unexpected element count");
            if (r.off + n * sizeof(float) > buf.size())
                parse_fail("checkpoint truncated while reading tensor data");
            if (!tensors[i]) input_fail("checkpoint: null tensor " + specs[i].name);
            std::memcpy(tensors[i], buf.data() + r.off, (size_t)n * sizeof(float));
            r.off += (size_t)n * sizeof(float);
        }
    });
}

}  // extern "C"
