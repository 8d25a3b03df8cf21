// srm_snapshot.cpp -- the reference's snapshot codec on the context state (SURVEY.md §8f
// row 4): checkpoint / resume of device-resident states in the reference's own file
// format (snapshot_io.cpp), byte for byte.
//
//   binary (snapshot_io.cpp:170-191): "SRMSNAP\0", u32 version 1, u64 header length,
//          header JSON, then per particle u32 id + the row's doubles (little endian)
//   text   (snapshot_io.cpp:150-167): header JSON line, column line, "id,v0,v1,...\n" rows
//          (std::to_chars shortest round-trip doubles)
// The header is built and dumped with nlohmann::json 3.11.3 -- the library and version
// the reference uses -- with the same keys and value types (snapshot_io.cpp:128-148), so
// the bytes equal the reference's snapshot_to_binary / snapshot_to_text (pinned in
// tests/test_snapshot.py).  Host code: the state crosses PCIe once per save / load.
#include <unistd.h>

#include <atomic>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../include/srm_b200.h"

namespace {

constexpr char kMagic[8] = {'S', 'R', 'M', 'S', 'N', 'A', 'P', '\0'};
constexpr std::uint32_t kVersion = 1;

struct Traits {
    const char* name;
    int dimension;
    const char* columns;
    int doubles;
};
constexpr Traits kDisk{"disk", 2, "id,x,y,r", 3};
constexpr Traits kSphere{"sphere", 3, "id,x,y,z,r", 4};
constexpr Traits kPlatelet{"spherodisk", 3, "id,x,y,z,nx,ny,nz,D,t", 8};

const Traits* traits(int dim, int shape) {
    if (shape == SRM_B200_PLATELET) return dim == 3 ? &kPlatelet : nullptr;
    return dim == 2 ? &kDisk : (dim == 3 ? &kSphere : nullptr);
}

struct IoFail {
    std::string what;
};

// snapshot_io.cpp:128-148 make_header + :30-41 params_to_json
std::string header_json(const Traits& tr, const double* box, int64_t n, const srm_b200_snapshot_meta& m) {
    nlohmann::json h = nlohmann::json::object();
    nlohmann::json b = nlohmann::json::array();
    for (int a = 0; a < tr.dimension; ++a) b.push_back(box[a]);
    h["box"] = std::move(b);
    h["count"] = static_cast<std::size_t>(n);
    h["dimension"] = tr.dimension;
    h["format"] = "srm-snapshot";
    h["iterations"] = static_cast<std::int64_t>(m.iteration_count);
    h["params"] = nlohmann::json{{"c_m", m.params.c_m},
                                 {"c_r", m.params.c_r},
                                 {"c_w", m.params.c_w},
                                 {"f_target", m.params.f_target},
                                 {"max_iterations", static_cast<std::int64_t>(m.params.max_iterations)},
                                 {"n_k", static_cast<int>(m.params.n_k)},
                                 {"n_l", static_cast<int>(m.params.n_l)},
                                 {"reorder_period", static_cast<int>(m.params.reorder_period)},
                                 {"seed", static_cast<std::uint64_t>(m.params.seed)}};
    h["seed"] = static_cast<std::uint64_t>(m.seed);
    h["shape"] = tr.name;
    h["version"] = kVersion;
    h["volume_fraction"] = m.volume_fraction;
    return h.dump();
}

// one particle's row values (snapshot_io.cpp:78-101 row_values)
void row(const Traits& tr, int64_t i, const double* pos, const double* r, const double* nrm, const double* D,
         const double* t, double* v) {
    if (tr.doubles == 8) {
        for (int a = 0; a < 3; ++a) {
            v[a] = pos[3 * i + a];
            v[3 + a] = nrm[3 * i + a];
        }
        v[6] = D[i];
        v[7] = t[i];
    } else {
        const int d = tr.dimension;
        for (int a = 0; a < d; ++a) v[a] = pos[d * i + a];
        v[d] = r[i];
    }
}

std::string encode(const Traits& tr, const double* box, int64_t n, const double* pos, const double* r,
                   const double* nrm, const double* D, const double* t, const int32_t* id,
                   const srm_b200_snapshot_meta& m, bool binary) {
    const std::string header = header_json(tr, box, n, m);
    std::string out;
    double v[8];
    if (binary) {
        out.reserve(64 + header.size() + static_cast<std::size_t>(n) * (4 + 8 * tr.doubles));
        out.append(kMagic, sizeof kMagic);
        const std::uint32_t ver = kVersion;
        out.append(reinterpret_cast<const char*>(&ver), 4);
        const std::uint64_t hlen = header.size();
        out.append(reinterpret_cast<const char*>(&hlen), 8);
        out += header;
        for (int64_t i = 0; i < n; ++i) {
            const std::uint32_t u = static_cast<std::uint32_t>(id[i]);
            out.append(reinterpret_cast<const char*>(&u), 4);
            row(tr, i, pos, r, nrm, D, t, v);
            out.append(reinterpret_cast<const char*>(v), 8 * tr.doubles);
        }
        return out;
    }
    out = header;
    out += '\n';
    out += tr.columns;
    out += '\n';
    char buf[32];
    for (int64_t i = 0; i < n; ++i) {
        auto res = std::to_chars(buf, buf + sizeof buf, static_cast<long long>(id[i]));
        out.append(buf, res.ptr);
        row(tr, i, pos, r, nrm, D, t, v);
        for (int c = 0; c < tr.doubles; ++c) {
            out += ',';
            res = std::to_chars(buf, buf + sizeof buf, v[c]);
            out.append(buf, res.ptr);
        }
        out += '\n';
    }
    return out;
}

// snapshot_io.cpp:392-414 write_file_atomic: a unique sibling, then rename
void write_atomic(const std::string& path, const std::string& content) {
    namespace fs = std::filesystem;
    const fs::path p(path);
    const fs::path dir = p.has_parent_path() ? p.parent_path() : fs::path(".");
    std::error_code ec;
    fs::create_directories(dir, ec);
    static std::atomic<std::uint64_t> counter{0};
    const fs::path tmp = dir / (p.filename().string() + ".tmp." + std::to_string(::getpid()) + "." +
                                std::to_string(counter.fetch_add(1)));
    {
        std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
        if (!out) throw IoFail{"cannot open for writing: " + tmp.string()};
        out.write(content.data(), static_cast<std::streamsize>(content.size()));
        if (!out) throw IoFail{"write failed: " + tmp.string()};
    }
    fs::rename(tmp, p, ec);
    if (ec) {
        fs::remove(tmp);
        throw IoFail{"rename failed for " + path + ": " + ec.message()};
    }
}

// a parsed file: header + row values (snapshot_io.cpp:353-381 parse_snapshot)
struct Parsed {
    const Traits* tr = nullptr;
    double box[3] = {1.0, 1.0, 1.0};
    int64_t n = 0;
    srm_b200_snapshot_meta meta{};
    std::vector<int32_t> id;
    std::vector<double> vals;  // n x tr->doubles
};

const nlohmann::json& require(const nlohmann::json& j, const char* key) {
    const auto it = j.find(key);
    if (it == j.end()) throw IoFail{std::string("snapshot header: missing key '") + key + "'"};
    return *it;
}

Parsed parse(const std::string& bytes, bool rows) {
    Parsed P;
    const bool binary = bytes.size() >= sizeof kMagic && std::memcmp(bytes.data(), kMagic, sizeof kMagic) == 0;
    const char* p = bytes.data();
    const char* end = bytes.data() + bytes.size();
    nlohmann::json h;
    try {
        if (binary) {
            p += sizeof kMagic;
            if (end - p < 12) throw IoFail{"snapshot: truncated binary header"};
            std::uint32_t ver;
            std::memcpy(&ver, p, 4);
            std::uint64_t hlen;
            std::memcpy(&hlen, p + 4, 8);
            p += 12;
            if (static_cast<std::uint64_t>(end - p) < hlen) throw IoFail{"snapshot: truncated binary header"};
            h = nlohmann::json::parse(p, p + hlen);
            p += hlen;
            if (ver != kVersion) throw IoFail{"snapshot: unsupported format version"};
        } else {
            const char* eol = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
            if (!eol) throw IoFail{"snapshot: missing header line"};
            h = nlohmann::json::parse(p, eol);
            p = eol + 1;
        }
    } catch (const nlohmann::json::exception& e) {
        throw IoFail{std::string("snapshot: bad header JSON: ") + e.what()};
    }
    try {
        const std::string shape = require(h, "shape").get<std::string>();
        const int dim = require(h, "dimension").get<int>();
        if (require(h, "version").get<std::uint32_t>() != kVersion) throw IoFail{"snapshot: unsupported format version"};
        if (require(h, "format").get<std::string>() != "srm-snapshot") throw IoFail{"snapshot: unrecognized format tag"};
        if (shape == "disk" && dim == 2) P.tr = &kDisk;
        else if (shape == "sphere" && dim == 3) P.tr = &kSphere;
        else if (shape == "spherodisk" && dim == 3) P.tr = &kPlatelet;
        else throw IoFail{"snapshot: unknown shape/dimension combination '" + shape + "'"};
        const auto& box = require(h, "box");
        if (!box.is_array() || box.size() != static_cast<std::size_t>(dim))
            throw IoFail{"snapshot header: box must list one length per axis"};
        for (int a = 0; a < dim; ++a) P.box[a] = box[a].get<double>();
        const auto& pj = require(h, "params");
        P.meta.params.c_m = require(pj, "c_m").get<double>();
        P.meta.params.c_r = require(pj, "c_r").get<double>();
        P.meta.params.c_w = require(pj, "c_w").get<double>();
        P.meta.params.f_target = require(pj, "f_target").get<double>();
        P.meta.params.max_iterations = require(pj, "max_iterations").get<std::int64_t>();
        P.meta.params.n_k = require(pj, "n_k").get<int>();
        P.meta.params.n_l = require(pj, "n_l").get<int>();
        P.meta.params.reorder_period = require(pj, "reorder_period").get<int>();
        P.meta.params.seed = require(pj, "seed").get<std::uint64_t>();
        P.meta.seed = require(h, "seed").get<std::uint64_t>();
        P.meta.iteration_count = require(h, "iterations").get<std::int64_t>();
        P.meta.volume_fraction = require(h, "volume_fraction").get<double>();
        P.n = static_cast<int64_t>(require(h, "count").get<std::size_t>());
    } catch (const nlohmann::json::exception& e) {
        throw IoFail{std::string("snapshot: bad header: ") + e.what()};
    }
    if (!rows) return P;
    const int nd = P.tr->doubles;
    P.id.resize(static_cast<size_t>(P.n));
    P.vals.resize(static_cast<size_t>(P.n) * nd);
    if (binary) {  // snapshot_io.cpp:286-306
        const std::size_t rb = 4 + 8 * static_cast<std::size_t>(nd);
        if (static_cast<std::size_t>(end - p) != rb * static_cast<std::size_t>(P.n))
            throw IoFail{"snapshot: binary payload size does not match count"};
        for (int64_t i = 0; i < P.n; ++i) {
            std::uint32_t u;
            std::memcpy(&u, p, 4);
            P.id[i] = static_cast<int32_t>(u);
            std::memcpy(&P.vals[i * nd], p + 4, 8 * nd);
            p += rb;
        }
        return P;
    }
    // text rows (snapshot_io.cpp:260-284): the column line, then id,v0,...\n per particle
    const std::size_t cl = std::strlen(P.tr->columns);
    if (static_cast<std::size_t>(end - p) < cl + 1 || std::memcmp(p, P.tr->columns, cl) != 0 || p[cl] != '\n')
        throw IoFail{"snapshot: column line does not match shape schema"};
    p += cl + 1;
    for (int64_t i = 0; i < P.n; ++i) {
        int v = 0;
        auto res = std::from_chars(p, end, v);
        if (res.ec != std::errc()) throw IoFail{"snapshot row: malformed integer"};
        p = res.ptr;
        P.id[i] = v;
        for (int c = 0; c < nd; ++c) {
            if (p == end || *p != ',') throw IoFail{"snapshot row: expected ','"};
            ++p;
            double d = 0.0;
            auto rd = std::from_chars(p, end, d);
            if (rd.ec != std::errc()) throw IoFail{"snapshot row: malformed number"};
            p = rd.ptr;
            P.vals[i * nd + c] = d;
        }
        if (p == end || *p != '\n') throw IoFail{"snapshot row: expected '\\n'"};
        ++p;
    }
    if (p != end) throw IoFail{"snapshot: trailing data after last row"};
    return P;
}

std::string read_file(const char* path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoFail{std::string("cannot open snapshot: ") + path};
    std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    if (in.bad()) throw IoFail{std::string("read failed: ") + path};
    return bytes;
}

thread_local std::string g_io_error;

template <typename F>
int io_guard(F&& f) {
    try {
        return f();
    } catch (const IoFail& e) {
        g_io_error = e.what;
        return SRM_B200_IO_ERROR;
    } catch (const std::bad_alloc&) {
        g_io_error = "out of host memory";
        return SRM_B200_IO_ERROR;
    } catch (const std::exception& e) {
        g_io_error = e.what();
        return SRM_B200_IO_ERROR;
    }
}

}  // namespace

extern "C" {

const char* srm_b200_io_error(void) { return g_io_error.c_str(); }

int srm_b200_snapshot_encode(int dim, int shape_kind, const double* box_lengths, int64_t n, const double* pos,
                             const double* radius, const double* normal, const double* diameter,
                             const double* thickness, const int32_t* id, const srm_b200_snapshot_meta* meta,
                             int binary, char* out, int64_t* len_inout) {
    const Traits* tr = traits(dim, shape_kind);
    if (!tr || n < 0 || !meta || !len_inout) return SRM_B200_INVALID;
    return io_guard([&]() -> int {
        const std::string s = encode(*tr, box_lengths, n, pos, radius, normal, diameter, thickness, id, *meta,
                                     binary != 0);
        const int64_t cap = *len_inout;
        *len_inout = static_cast<int64_t>(s.size());
        if (out) {
            if (cap < static_cast<int64_t>(s.size())) return SRM_B200_INVALID;
            std::memcpy(out, s.data(), s.size());
        }
        return SRM_B200_OK;
    });
}

int srm_b200_save_snapshot(srm_b200_ctx* ctx, const char* path, const srm_b200_snapshot_meta* meta, int binary) {
    int dim = 0, shape = 0;
    double box[3];
    if (!ctx || !path || !meta || srm_b200_describe(ctx, &dim, &shape, box) != SRM_B200_OK) return SRM_B200_INVALID;
    const Traits* tr = traits(dim, shape);
    if (!tr) return SRM_B200_INVALID;
    const int64_t n = srm_b200_count(ctx);
    std::vector<double> pos(static_cast<size_t>(n) * dim + 1), r(n + 1), nrm(3 * n + 3), D(n + 1), t(n + 1);
    std::vector<int32_t> id(n + 1);
    const int st = shape == SRM_B200_PLATELET
                       ? srm_b200_download_platelets(ctx, pos.data(), nrm.data(), D.data(), t.data(), id.data())
                       : srm_b200_download(ctx, pos.data(), r.data(), id.data());
    if (st != SRM_B200_OK) return st;
    return io_guard([&]() -> int {
        write_atomic(path, encode(*tr, box, n, pos.data(), r.data(), nrm.data(), D.data(), t.data(), id.data(), *meta,
                                  binary != 0));
        return SRM_B200_OK;
    });
}

int srm_b200_snapshot_info(const char* path, int* dim, int* shape_kind, int64_t* count, double* box_lengths,
                           srm_b200_snapshot_meta* meta) {
    if (!path) return SRM_B200_INVALID;
    return io_guard([&]() -> int {
        const Parsed P = parse(read_file(path), false);
        if (dim) *dim = P.tr->dimension;
        if (shape_kind) *shape_kind = P.tr == &kPlatelet ? SRM_B200_PLATELET : SRM_B200_SPHERE;
        if (count) *count = P.n;
        if (box_lengths)
            for (int a = 0; a < P.tr->dimension; ++a) box_lengths[a] = P.box[a];
        if (meta) *meta = P.meta;
        return SRM_B200_OK;
    });
}

int srm_b200_load_snapshot(srm_b200_ctx* ctx, const char* path) {
    int dim = 0, shape = 0;
    double box[3];
    if (!ctx || !path || srm_b200_describe(ctx, &dim, &shape, box) != SRM_B200_OK) return SRM_B200_INVALID;
    Parsed P;
    const int st = io_guard([&]() -> int {
        P = parse(read_file(path), true);
        return SRM_B200_OK;
    });
    if (st != SRM_B200_OK) return st;
    if (P.tr != traits(dim, shape)) {
        g_io_error = "snapshot: shape/dimension differ from the context's";
        return SRM_B200_INVALID;
    }
    for (int a = 0; a < dim; ++a)
        if (P.box[a] != box[a]) {
            g_io_error = "snapshot: box differs from the context's";
            return SRM_B200_INVALID;
        }
    const int64_t n = P.n;
    const int nd = P.tr->doubles;
    if (shape == SRM_B200_PLATELET) {
        std::vector<double> pos(3 * n + 3), nrm(3 * n + 3), D(n + 1), t(n + 1);
        for (int64_t i = 0; i < n; ++i) {
            for (int a = 0; a < 3; ++a) {
                pos[3 * i + a] = P.vals[i * nd + a];
                nrm[3 * i + a] = P.vals[i * nd + 3 + a];
            }
            D[i] = P.vals[i * nd + 6];
            t[i] = P.vals[i * nd + 7];
        }
        return srm_b200_upload_platelets(ctx, n, pos.data(), nrm.data(), D.data(), t.data(), P.id.data());
    }
    std::vector<double> pos(static_cast<size_t>(n) * dim + 1), r(n + 1);
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < dim; ++a) pos[i * dim + a] = P.vals[i * nd + a];
        r[i] = P.vals[i * nd + dim];
    }
    return srm_b200_upload(ctx, n, pos.data(), r.data(), P.id.data());
}

}  // extern "C"
