// rtk_host.cpp — host-side harness utilities behind the C-ABI:
//   * the reference's seeded input generators (datagen.hpp:18-140), so a report produced here
//     runs on exactly the inputs `rtk bench` / `rtk gen` produce on the CPU side;
//   * the result checksum of `rtk bench` (FNV-1a over (value bits, u64 index), rtk_cli.cpp:100-115);
//   * the RTK1 single-array and RTKB batch container formats (io.hpp:1-8, io.cpp:25-110).
// No device code: these are the harness around the hot path, not the hot path.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/rtk_c.h"
#include "rtk_guard.h"
#include "rtk_kernels.h"
#include "rtk_philox.h"

using rtk_b200::Error;
using rtk_b200::guarded;

namespace {

Error bad(const std::string& m) { return Error{RTK_INVALID_ARGUMENT, m}; }
Error io_error(const std::string& m) { return Error{RTK_IO_ERROR, m}; }

// DistributionSpec::validate (datagen.hpp:27-48)
void check_spec(const rtk_dist* d) {
    if (!d) throw bad("distribution: null spec");
    if (d->n == 0) throw bad("distribution: n must be positive");
    switch (d->kind) {
        case RTK_DIST_UNIFORM:
            if (!(d->a < d->b)) throw bad("uniform: requires a < b");
            break;
        case RTK_DIST_NORMAL:
            if (!(d->b > 0)) throw bad("normal: requires sigma > 0");
            break;
        case RTK_DIST_ZIPF:
            if (!(d->s > 1.0)) throw bad("zipf: requires s > 1");
            break;
        case RTK_DIST_PEAKED:
            if (!(d->mass > 0.0 && d->mass < 1.0)) throw bad("peaked: mass must be in (0, 1)");
            if (d->modes == 0 || d->modes >= d->n) throw bad("peaked: modes must be in [1, n)");
            break;
        default:
            throw bad("distribution: unknown kind");
    }
}

// rank-law masses r^-s / H_n in rank order, rounded to f32 (datagen.hpp:55-66)
std::vector<float> rank_law(uint64_t n, double s) {
    std::vector<double> w(n);
    double h = 0.0;
    for (uint64_t r = 0; r < n; ++r) h += (w[r] = std::pow(static_cast<double>(r + 1), -s));
    std::vector<float> f(n);
    for (uint64_t r = 0; r < n; ++r) f[r] = static_cast<float>(w[r] / h);
    return f;
}

template <typename Dist>
void fill_f32(float* out, uint64_t n, Dist dist, std::mt19937_64& rng) {
    for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<float>(dist(rng));
}

void generate_f32(const rtk_dist* d, float* out) {
    std::mt19937_64 rng(d->seed);
    const uint64_t n = d->n;
    if (d->kind == RTK_DIST_UNIFORM) {
        fill_f32(out, n, std::uniform_real_distribution<double>(d->a, d->b), rng);
    } else if (d->kind == RTK_DIST_NORMAL) {
        fill_f32(out, n, std::normal_distribution<double>(d->a, d->b), rng);
    } else if (d->kind == RTK_DIST_ZIPF) {
        const std::vector<float> m = rank_law(n, d->s);
        std::copy(m.begin(), m.end(), out);
        std::shuffle(out, out + n, rng);
    } else {  // peaked: `modes` modes share `mass`, the rest uniform around the residual mean
        const double mode = d->mass / d->modes;
        const double rest = (1.0 - d->mass) / static_cast<double>(n - d->modes);
        fill_f32(out, n, std::uniform_real_distribution<double>(rest * 0.5, rest * 1.5), rng);
        for (uint32_t m = 0; m < d->modes; ++m) out[m] = static_cast<float>(mode);
        std::shuffle(out, out + n, rng);
    }
}

void generate_u32(const rtk_dist* d, uint32_t* out) {
    std::mt19937_64 rng(d->seed);
    const uint64_t n = d->n;
    if (d->kind == RTK_DIST_UNIFORM) {
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(rng());
    } else if (d->kind == RTK_DIST_NORMAL) {
        std::normal_distribution<double> dist(2147483648.0, 536870912.0);
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(std::clamp(dist(rng), 0.0, 4294967295.0));
    } else if (d->kind == RTK_DIST_ZIPF) {  // masses in 30-bit fixed point
        const std::vector<float> m = rank_law(n, d->s);
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(m[i] * 1073741824.0f);
        std::shuffle(out, out + n, rng);
    } else {
        throw bad("peaked distribution is defined for f32 only");
    }
}

size_t elem_size(int dtype) {
    if (dtype == RTK_F32 || dtype == RTK_U32) return 4;
    if (dtype == RTK_F16 || dtype == RTK_BF16) return 2;
    throw bad("unknown dtype code " + std::to_string(dtype));
}

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const std::string& p, const char* mode) : f(std::fopen(p.c_str(), mode)), path(p) {}
    ~File() {
        if (f) std::fclose(f);
    }
    void get(void* dst, size_t bytes) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw io_error(path + ": truncated file");
    }
    void put(const void* src, size_t bytes) {
        if (bytes && std::fwrite(src, 1, bytes, f) != bytes) throw io_error(path + ": write failed");
    }
};

const char kRtk1[4] = {'R', 'T', 'K', '1'};
const char kRtkb[4] = {'R', 'T', 'K', 'B'};

}  // namespace

extern "C" {

int rtk_generate(const rtk_dist* spec, int dtype, void* out) {
    return guarded([&] {
        check_spec(spec);
        if (!out) throw bad("generate: null output");
        if (dtype == RTK_F32) generate_f32(spec, static_cast<float*>(out));
        else if (dtype == RTK_U32) generate_u32(spec, static_cast<uint32_t*>(out));
        else throw bad("generate: dtype must be F32 or U32 (datagen.hpp:68-140)");
    });
}

uint64_t rtk_result_checksum(const void* values, int dtype, const uint64_t* indices, uint64_t k) {
    // FNV-1a 64 over (value bytes, u64 index bytes) per element, little-endian
    uint64_t h = 14695981039346656037ull;
    const size_t vb = (dtype == RTK_F16 || dtype == RTK_BF16) ? 2 : 4;
    const unsigned char* v = static_cast<const unsigned char*>(values);
    for (uint64_t i = 0; i < k; ++i) {
        for (size_t b = 0; b < vb; ++b) h = (h ^ v[i * vb + b]) * 1099511628211ull;
        unsigned char ib[8];
        std::memcpy(ib, indices + i, 8);
        for (unsigned char c : ib) h = (h ^ c) * 1099511628211ull;
    }
    return h;
}

int rtk_write_dataset(const char* path, int dtype, const void* data, uint64_t n) {
    return guarded([&] {
        if (!path || (n && !data)) throw bad("write_dataset: null argument");
        const size_t eb = elem_size(dtype);
        File f(path, "wb");
        if (!f.f) throw io_error(std::string(path) + ": cannot open for writing");
        const uint8_t code = static_cast<uint8_t>(dtype);
        f.put(kRtk1, 4);
        f.put(&code, 1);
        f.put(&n, 8);
        f.put(data, n * eb);
    });
}

int rtk_read_dataset(const char* path, int* dtype, uint64_t* n, void* out, uint64_t capacity) {
    return guarded([&] {
        if (!path || !dtype || !n) throw bad("read_dataset: null argument");
        File f(path, "rb");
        if (!f.f) throw io_error(std::string(path) + ": cannot open");
        char magic[4];
        f.get(magic, 4);
        if (std::memcmp(magic, kRtk1, 4) != 0) throw io_error(std::string(path) + ": bad magic, not an RTK1 dataset");
        uint8_t code = 0;
        uint64_t count = 0;
        f.get(&code, 1);
        f.get(&count, 8);
        if (code > RTK_BF16) throw io_error(std::string(path) + ": unknown dtype code " + std::to_string(code));
        *dtype = code;
        *n = count;
        if (!out) return;  // size query
        if (capacity < count) throw bad("read_dataset: output capacity " + std::to_string(capacity) + " < " +
                                        std::to_string(count));
        f.get(out, count * elem_size(code));
    });
}

int rtk_write_batch(const char* path, const uint64_t* lengths, uint32_t tasks, const void* payload,
                    uint64_t payload_bytes) {
    return guarded([&] {
        if (!path || (tasks && !lengths) || (payload_bytes && !payload)) throw bad("write_batch: null argument");
        File f(path, "wb");
        if (!f.f) throw io_error(std::string(path) + ": cannot open for writing");
        f.put(kRtkb, 4);
        f.put(&tasks, 4);
        f.put(lengths, 8ull * tasks);
        f.put(payload, payload_bytes);
    });
}

int rtk_read_batch(const char* path, uint32_t* tasks, uint64_t* payload_bytes, uint64_t* lengths,
                   void* payload) {
    return guarded([&] {
        if (!path || !tasks || !payload_bytes) throw bad("read_batch: null argument");
        File f(path, "rb");
        if (!f.f) throw io_error(std::string(path) + ": cannot open");
        char magic[4];
        f.get(magic, 4);
        if (std::memcmp(magic, kRtkb, 4) != 0) throw io_error(std::string(path) + ": bad magic, not an RTKB batch");
        uint32_t count = 0;
        f.get(&count, 4);
        std::fseek(f.f, 0, SEEK_END);
        const long end = std::ftell(f.f);
        const long header = 8 + 8l * count;
        if (end < header) throw io_error(std::string(path) + ": truncated file");
        *tasks = count;
        *payload_bytes = static_cast<uint64_t>(end - header);
        if (!lengths && !payload) return;  // size query
        std::fseek(f.f, 8, SEEK_SET);
        if (lengths) f.get(lengths, 8ull * count);
        else std::fseek(f.f, header, SEEK_SET);
        if (payload) f.get(payload, *payload_bytes);
    });
}

}  // extern "C"

extern "C" int rtk_generate_philox(float* d_out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b,
                                   void* stream) {
    return guarded([&] {
        if (!d_out && n) throw bad("philox: null output");
        if (!(a < b)) throw bad("uniform: requires a < b");
        rtk_b200::launch_philox_uniform(d_out, n, seed, offset, a, b, static_cast<cudaStream_t>(stream));
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw Error{RTK_CUDA_ERROR, std::string("philox launch: ") + cudaGetErrorString(e)};
    });
}

extern "C" int rtk_generate_philox_host(float* out, uint64_t n, uint64_t seed, uint64_t offset, float a, float b) {
    return guarded([&] {
        if (!out && n) throw bad("philox: null output");
        if (!(a < b)) throw bad("uniform: requires a < b");
        const float span = b - a;
        uint64_t g = offset;
        for (uint64_t j = 0; j < n;) {
            uint32_t w[4];
            rtk_b200::philox_block(seed, g >> 2, w);
            for (uint32_t q = static_cast<uint32_t>(g & 3); q < 4 && j < n; ++q, ++j, ++g)
                out[j] = rtk_b200::philox_uniform(w[q], a, span);
        }
    });
}
