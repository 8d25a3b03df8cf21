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
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>

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

// Crash-safe save (the reference's write_file_atomic contract, snapshot_io.cpp:392-414:
// a reader sees the old file or the complete new one, never a torn write).  Done with
// POSIX calls: a mkstemp(3) temporary next to the target, a full write(2) loop, fsync(2),
// then rename(2) over the target (atomic within one filesystem).
void write_atomic(const std::string& path, const std::string& content) {
    namespace fs = std::filesystem;
    const fs::path target(path);
    const fs::path parent = target.has_parent_path() ? target.parent_path() : fs::path(".");
    std::error_code mk;
    fs::create_directories(parent, mk);
    std::string templ = (parent / ("." + target.filename().string() + ".partial-XXXXXX")).string();
    const int fd = ::mkstemp(templ.data());
    if (fd < 0) throw IoFail{"snapshot save: no temporary file beside " + path + ": " + std::strerror(errno)};
    auto abandon = [&](const std::string& what) {
        const int e = errno;
        ::close(fd);
        ::unlink(templ.c_str());
        throw IoFail{"snapshot save: " + what + " " + templ + ": " + std::strerror(e)};
    };
    const char* p = content.data();
    size_t left = content.size();
    while (left > 0) {
        const ssize_t w = ::write(fd, p, left);
        if (w < 0) {
            if (errno == EINTR) continue;
            abandon("write to");
        }
        p += w;
        left -= static_cast<size_t>(w);
    }
    if (::fchmod(fd, 0644) != 0 || ::fsync(fd) != 0) abandon("flush of");
    if (::close(fd) != 0) {
        ::unlink(templ.c_str());
        throw IoFail{"snapshot save: close of " + templ + " failed"};
    }
    if (::rename(templ.c_str(), path.c_str()) != 0) {
        const int e = errno;
        ::unlink(templ.c_str());
        throw IoFail{"snapshot save: cannot move " + templ + " to " + path + ": " + std::strerror(e)};
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

[[noreturn]] void bad_file(const std::string& why) { throw IoFail{"snapshot load: " + why}; }

const nlohmann::json& field(const nlohmann::json& obj, const char* name) {
    const auto it = obj.find(name);
    if (it == obj.end()) bad_file(std::string("header has no '") + name + "' entry");
    return *it;
}

// a read position over the file bytes
struct Cursor {
    const char* p;
    const char* end;
    size_t left() const { return static_cast<size_t>(end - p); }
    template <typename T>
    T raw() {  // little-endian fixed-width field
        if (left() < sizeof(T)) bad_file("file ends inside the binary header");
        T v;
        std::memcpy(&v, p, sizeof(T));
        p += sizeof(T);
        return v;
    }
    void expect(char ch, const char* what) {
        if (p == end || *p != ch) bad_file(std::string("row ") + what);
        ++p;
    }
    template <typename T>
    T number(const char* what) {
        T v{};
        const auto r = std::from_chars(p, end, v);
        if (r.ec != std::errc()) bad_file(std::string("row has an unreadable ") + what);
        p = r.ptr;
        return v;
    }
};

// the JSON header: after the magic + version + length in the binary layout
// (snapshot_io.cpp:170-191), or the first line of the text layout (snapshot_io.cpp:150-167)
nlohmann::json read_header(Cursor& c, bool binary) {
    try {
        if (binary) {
            c.p += sizeof kMagic;
            const std::uint32_t version = c.raw<std::uint32_t>();
            const std::uint64_t len = c.raw<std::uint64_t>();
            if (c.left() < len) bad_file("file ends inside the binary header");
            nlohmann::json h = nlohmann::json::parse(c.p, c.p + len);
            c.p += len;
            if (version != kVersion) bad_file("format version " + std::to_string(version) + " is not supported");
            return h;
        }
        const char* nl = static_cast<const char*>(std::memchr(c.p, '\n', c.left()));
        if (!nl) bad_file("no header line");
        nlohmann::json h = nlohmann::json::parse(c.p, nl);
        c.p = nl + 1;
        return h;
    } catch (const nlohmann::json::exception& e) {
        bad_file(std::string("header is not valid JSON (") + e.what() + ")");
    }
}

// header keys and types as the reference writes them (snapshot_io.cpp:128-148)
void read_meta(const nlohmann::json& h, Parsed& P) {
    try {
        const std::string shape = field(h, "shape").get<std::string>();
        const int dim = field(h, "dimension").get<int>();
        if (field(h, "version").get<std::uint32_t>() != kVersion) bad_file("header names an unsupported version");
        if (field(h, "format").get<std::string>() != "srm-snapshot") bad_file("header is not an srm-snapshot");
        for (const Traits* t : {&kDisk, &kSphere, &kPlatelet})
            if (shape == t->name && dim == t->dimension) P.tr = t;
        if (!P.tr) bad_file("no shape '" + shape + "' in dimension " + std::to_string(dim));
        const auto& box = field(h, "box");
        if (!box.is_array() || box.size() != static_cast<std::size_t>(dim))
            bad_file("box lengths do not match the dimension");
        for (int a = 0; a < dim; ++a) P.box[a] = box[a].get<double>();
        const auto& pj = field(h, "params");
        srm_b200_params& q = P.meta.params;
        q.c_m = field(pj, "c_m").get<double>();
        q.c_r = field(pj, "c_r").get<double>();
        q.c_w = field(pj, "c_w").get<double>();
        q.f_target = field(pj, "f_target").get<double>();
        q.max_iterations = field(pj, "max_iterations").get<std::int64_t>();
        q.n_k = field(pj, "n_k").get<int>();
        q.n_l = field(pj, "n_l").get<int>();
        q.reorder_period = field(pj, "reorder_period").get<int>();
        q.seed = field(pj, "seed").get<std::uint64_t>();
        P.meta.seed = field(h, "seed").get<std::uint64_t>();
        P.meta.iteration_count = field(h, "iterations").get<std::int64_t>();
        P.meta.volume_fraction = field(h, "volume_fraction").get<double>();
        P.n = static_cast<int64_t>(field(h, "count").get<std::size_t>());
    } catch (const nlohmann::json::exception& e) {
        bad_file(std::string("header has a field of the wrong type (") + e.what() + ")");
    }
}

Parsed parse(const std::string& bytes, bool rows) {
    Parsed P;
    Cursor c{bytes.data(), bytes.data() + bytes.size()};
    const bool binary = c.left() >= sizeof kMagic && std::memcmp(c.p, kMagic, sizeof kMagic) == 0;
    read_meta(read_header(c, binary), P);
    if (!rows) return P;
    const int nd = P.tr->doubles;
    P.id.resize(static_cast<size_t>(P.n));
    P.vals.resize(static_cast<size_t>(P.n) * nd);
    if (binary) {  // fixed-width records: u32 id + nd doubles (snapshot_io.cpp:286-306)
        const std::size_t width = 4 + 8 * static_cast<std::size_t>(nd);
        if (c.left() != width * static_cast<std::size_t>(P.n)) bad_file("record block size disagrees with the count");
        for (int64_t i = 0; i < P.n; ++i) {
            P.id[i] = static_cast<int32_t>(c.raw<std::uint32_t>());
            std::memcpy(&P.vals[i * nd], c.p, 8 * static_cast<size_t>(nd));
            c.p += 8 * nd;
        }
        return P;
    }
    // text (snapshot_io.cpp:260-284): the column line, then one "id,v0,...,vk" line per particle
    const std::string cols = std::string(P.tr->columns) + "\n";
    if (c.left() < cols.size() || std::memcmp(c.p, cols.data(), cols.size()) != 0)
        bad_file("column line is not the one of this shape");
    c.p += cols.size();
    for (int64_t i = 0; i < P.n; ++i) {
        P.id[i] = c.number<int>("id");
        for (int k = 0; k < nd; ++k) {
            c.expect(',', "is missing a ','");
            P.vals[i * nd + k] = c.number<double>("value");
        }
        c.expect('\n', "does not end with a newline");
    }
    if (c.left() != 0) bad_file("bytes after the last row");
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
