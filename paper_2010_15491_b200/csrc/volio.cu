// .volhdr / .vol volume I/O (reference src/volume_io.cpp, include/volsr/volume_io.hpp):
// the data format on either side of the solver path.  Header: text lines
// dims=m,n,s / dtype=f32|f64 / order=lex; payload: raw little-endian scalars in
// lexicographic order (axis 1 fastest).
//
// Host entry points restate the reference's load_volume / save_volume.  The
// `_d` entry points stream the payload between the file and device memory in
// 32 MB chunks through two pinned buffers: the file read (or write) of one
// chunk overlaps the PCIe copy of the other, an f32 payload crosses PCIe as
// f32 and is widened (or narrowed) on the device, and the finiteness check of
// the reference (first non-finite flat index) runs on the device.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/vsr.h"
#include "vsr_common.cuh"

namespace vsr_capi {
cudaStream_t stream_of(vsr_ctx* ctx);
int device_of(vsr_ctx* ctx);
int guard_call(const std::function<void()>& f);
}  // namespace vsr_capi

namespace vsr {
namespace {

bool ends_with(const std::string& s, const std::string& suffix) {
    return s.size() >= suffix.size() && s.compare(s.size() - suffix.size(), suffix.size(), suffix) == 0;
}

std::string strip_ext(const std::string& path) {
    if (ends_with(path, ".volhdr")) return path.substr(0, path.size() - 7);
    if (ends_with(path, ".vol")) return path.substr(0, path.size() - 4);
    return path;
}

std::string dims_str(const size_t d[3]) {
    return std::to_string(d[0]) + "x" + std::to_string(d[1]) + "x" + std::to_string(d[2]);
}

struct Header {
    size_t dims[3] = {0, 0, 0};
    int dtype = VSR_DTYPE_F64;
};

// volume_io.cpp:17-25
void parse_dims(const std::string& value, const std::string& path, size_t d[3]) {
    char c1 = 0, c2 = 0;
    std::istringstream is(value);
    if (!(is >> d[0] >> c1 >> d[1] >> c2 >> d[2]) || c1 != ',' || c2 != ',' || !(is >> std::ws).eof())
        throw io_error(path + ": malformed dims '" + value + "'");
    if (d[0] * d[1] * d[2] == 0) throw io_error(path + ": zero-sized dims '" + value + "'");
}

// volume_io.cpp:65-106 (header part of load_volume)
Header read_header(const std::string& base) {
    const std::string hdr_path = base + ".volhdr";
    std::ifstream hdr(hdr_path);
    if (!hdr) throw io_error("load_volume: cannot open " + hdr_path);
    bool have_dims = false, have_dtype = false, have_order = false;
    Header h;
    std::string line;
    while (std::getline(hdr, line)) {
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos) throw io_error(hdr_path + ": malformed line '" + line + "'");
        const std::string key = line.substr(0, eq), value = line.substr(eq + 1);
        if (key == "dims") {
            if (have_dims) throw io_error(hdr_path + ": duplicate dims");
            parse_dims(value, hdr_path, h.dims);
            have_dims = true;
        } else if (key == "dtype") {
            if (have_dtype) throw io_error(hdr_path + ": duplicate dtype");
            if (value == "f32")
                h.dtype = VSR_DTYPE_F32;
            else if (value == "f64")
                h.dtype = VSR_DTYPE_F64;
            else
                throw io_error(hdr_path + ": unsupported dtype '" + value + "'");
            have_dtype = true;
        } else if (key == "order") {
            if (value != "lex") throw io_error(hdr_path + ": unsupported order '" + value + "'");
            have_order = true;
        } else {
            throw io_error(hdr_path + ": unknown key '" + key + "'");
        }
    }
    if (!have_dims || !have_dtype || !have_order)
        throw io_error(hdr_path + ": incomplete header (need dims, dtype, order)");
    return h;
}

size_t count_of(const size_t d[3]) { return d[0] * d[1] * d[2]; }

// opens the payload and checks its length against the header (volume_io.cpp:108-116)
FILE* open_payload(const std::string& base, const Header& h) {
    const std::string raw_path = base + ".vol";
    FILE* f = std::fopen(raw_path.c_str(), "rb");
    if (!f) throw io_error("load_volume: cannot open " + raw_path);
    std::fseek(f, 0, SEEK_END);
    const auto actual = static_cast<uint64_t>(std::ftell(f));
    std::fseek(f, 0, SEEK_SET);
    const size_t scalar = h.dtype == VSR_DTYPE_F32 ? sizeof(float) : sizeof(double);
    const uint64_t expected = static_cast<uint64_t>(count_of(h.dims)) * scalar;
    if (actual != expected) {
        std::fclose(f);
        throw io_error(raw_path + ": payload is " + std::to_string(actual) + " bytes, expected " +
                       std::to_string(expected) + " for dims " + dims_str(h.dims));
    }
    return f;
}

void write_header(const std::string& base, const size_t d[3], int dtype) {
    std::ofstream hdr(base + ".volhdr");
    if (!hdr) throw io_error("save_volume: cannot open " + base + ".volhdr for writing");
    hdr << "dims=" << d[0] << "," << d[1] << "," << d[2] << "\n"
        << "dtype=" << (dtype == VSR_DTYPE_F32 ? "f32" : "f64") << "\n"
        << "order=lex\n";
    if (!hdr) throw io_error("save_volume: failed writing " + base + ".volhdr");
}

void check_dtype(int dtype) {
    if (dtype != VSR_DTYPE_F32 && dtype != VSR_DTYPE_F64)
        throw std::invalid_argument("save_volume: dtype must be VSR_DTYPE_F32 or VSR_DTYPE_F64");
}

// ------------------------------------------------------------------ device side
constexpr size_t kChunk = 32u << 20;  // bytes per streamed chunk

__global__ void widen_kernel(const float* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}

__global__ void narrow_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

// first non-finite flat index (integer atomicMin: order-independent result)
__global__ void first_nonfinite_kernel(const double* __restrict__ v, long long n, unsigned long long* bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) atomicMin(bad, (unsigned long long)i);
}

unsigned grid_for(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16); }

unsigned long long device_first_nonfinite(const double* v, long long n, cudaStream_t st) {
    unsigned long long* bad = nullptr;
    VSR_CUDA(cudaMallocAsync(&bad, sizeof(unsigned long long), st));
    VSR_CUDA(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), st));
    first_nonfinite_kernel<<<grid_for(n), 256, 0, st>>>(v, n, bad);
    VSR_LAUNCH_CHECK();
    unsigned long long h = 0;
    VSR_CUDA(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    VSR_CUDA(cudaFreeAsync(bad, st));
    VSR_CUDA(cudaStreamSynchronize(st));
    return h;
}

struct Pinned {
    void* p[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    Pinned() {
        for (int i = 0; i < 2; ++i) {
            VSR_CUDA(cudaMallocHost(&p[i], kChunk));
            VSR_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
    }
    ~Pinned() {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
            if (p[i]) cudaFreeHost(p[i]);
        }
    }
};

struct DevGuard {
    int prev = 0, want;
    explicit DevGuard(int dev) : want(dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev != want) cudaSetDevice(prev);
    }
};

}  // namespace
}  // namespace vsr

using namespace vsr;

extern "C" {

int vsr_volume_header(const char* path, size_t dims_out[3], int* dtype_out) {
    return vsr_capi::guard_call([&] {
        const Header h = read_header(strip_ext(path));
        for (int a = 0; a < 3; ++a) dims_out[a] = h.dims[a];
        if (dtype_out) *dtype_out = h.dtype;
    });
}

// volume_io.cpp:61-131 (load_volume), into a caller buffer of `count` doubles
int vsr_load_volume(const char* path, double* out, size_t count) {
    return vsr_capi::guard_call([&] {
        const std::string base = strip_ext(path);
        const Header h = read_header(base);
        const size_t n = count_of(h.dims);
        if (n != count)
            throw shape_error("load_volume: volume has " + std::to_string(n) + " values (dims " + dims_str(h.dims) +
                              "), buffer holds " + std::to_string(count));
        FILE* f = open_payload(base, h);
        size_t got;
        if (h.dtype == VSR_DTYPE_F64) {
            got = std::fread(out, sizeof(double), n, f);
        } else {
            std::vector<float> buf(n);
            got = std::fread(buf.data(), sizeof(float), n, f);
            for (size_t p = 0; p < n; ++p) out[p] = (double)buf[p];
        }
        std::fclose(f);
        if (got != n) throw io_error(base + ".vol: short read");
        for (size_t p = 0; p < n; ++p)
            if (!std::isfinite(out[p]))
                throw io_error(base + ".vol: non-finite value at flat index " + std::to_string(p));
    });
}

// volume_io.cpp:34-57 (save_volume)
int vsr_save_volume(const char* path, const size_t dims[3], const double* v, int dtype) {
    return vsr_capi::guard_call([&] {
        check_dtype(dtype);
        const size_t n = count_of(dims);
        for (size_t p = 0; p < n; ++p)
            if (!std::isfinite(v[p]))
                throw numeric_error("save_volume: non-finite value at flat index " + std::to_string(p));
        const std::string base = strip_ext(path);
        write_header(base, dims, dtype);
        FILE* f = std::fopen((base + ".vol").c_str(), "wb");
        if (!f) throw io_error("save_volume: cannot open " + base + ".vol for writing");
        size_t put;
        if (dtype == VSR_DTYPE_F64) {
            put = std::fwrite(v, sizeof(double), n, f);
        } else {
            std::vector<float> buf(n);
            for (size_t p = 0; p < n; ++p) buf[p] = (float)v[p];
            put = std::fwrite(buf.data(), sizeof(float), n, f);
        }
        const bool ok = put == n && std::fclose(f) == 0;
        if (!ok) throw io_error("save_volume: failed writing " + base + ".vol");
    });
}

// load_volume streamed into device memory (dev_out: `count` doubles on the
// context's device).  Chunk k is read from the file into pinned buffer k % 2
// while chunk k - 1's H2D copy (and, for f32, its widening) runs.
int vsr_load_volume_d(vsr_ctx* ctx, const char* path, double* dev_out, size_t count) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        cudaStream_t st = vsr_capi::stream_of(ctx);
        const std::string base = strip_ext(path);
        const Header h = read_header(base);
        const size_t n = count_of(h.dims);
        if (n != count)
            throw shape_error("load_volume: volume has " + std::to_string(n) + " values (dims " + dims_str(h.dims) +
                              "), buffer holds " + std::to_string(count));
        const bool f32 = h.dtype == VSR_DTYPE_F32;
        const size_t scalar = f32 ? sizeof(float) : sizeof(double);
        const size_t per = kChunk / scalar;  // values per chunk
        FILE* f = open_payload(base, h);
        float* stage = nullptr;  // f32: device staging of the narrow payload
        try {
            Pinned pin;
            if (f32) VSR_CUDA(cudaMallocAsync(&stage, std::min(n, 2 * per) * sizeof(float), st));
            size_t k = 0;
            for (size_t off = 0; off < n; off += per, ++k) {
                const int b = (int)(k & 1);
                const size_t len = std::min(per, n - off);
                VSR_CUDA(cudaEventSynchronize(pin.done[b]));  // buffer b's previous copy has left
                if (std::fread(pin.p[b], scalar, len, f) != len) throw io_error(base + ".vol: short read");
                if (f32) {
                    float* sb = stage + (size_t)b * per;
                    VSR_CUDA(cudaMemcpyAsync(sb, pin.p[b], len * sizeof(float), cudaMemcpyHostToDevice, st));
                    widen_kernel<<<grid_for((long long)len), 256, 0, st>>>(sb, dev_out + off, (long long)len);
                    VSR_LAUNCH_CHECK();
                } else {
                    VSR_CUDA(cudaMemcpyAsync(dev_out + off, pin.p[b], len * sizeof(double), cudaMemcpyHostToDevice,
                                             st));
                }
                VSR_CUDA(cudaEventRecord(pin.done[b], st));
            }
            if (stage) VSR_CUDA(cudaFreeAsync(stage, st));
            stage = nullptr;
        } catch (...) {
            std::fclose(f);
            if (stage) cudaFreeAsync(stage, st);
            throw;
        }
        std::fclose(f);
        const unsigned long long bad = device_first_nonfinite(dev_out, (long long)n, st);
        if (bad != ~0ull) throw io_error(base + ".vol: non-finite value at flat index " + std::to_string(bad));
    });
}

// save_volume from device memory: the finiteness check runs on the device,
// then chunk k's D2H copy (f32: narrowed on the device first) overlaps the
// file write of chunk k - 1.
int vsr_save_volume_d(vsr_ctx* ctx, const char* path, const size_t dims[3], const double* dev_in, int dtype) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        cudaStream_t st = vsr_capi::stream_of(ctx);
        check_dtype(dtype);
        const size_t n = count_of(dims);
        const unsigned long long bad = device_first_nonfinite(dev_in, (long long)n, st);
        if (bad != ~0ull) throw numeric_error("save_volume: non-finite value at flat index " + std::to_string(bad));
        const std::string base = strip_ext(path);
        write_header(base, dims, dtype);
        FILE* f = std::fopen((base + ".vol").c_str(), "wb");
        if (!f) throw io_error("save_volume: cannot open " + base + ".vol for writing");
        const bool f32 = dtype == VSR_DTYPE_F32;
        const size_t scalar = f32 ? sizeof(float) : sizeof(double);
        const size_t per = kChunk / scalar;
        float* stage = nullptr;
        bool ok = true;
        try {
            Pinned pin;
            if (f32) VSR_CUDA(cudaMallocAsync(&stage, std::min(n, 2 * per) * sizeof(float), st));
            size_t pending_len = 0;
            int pending_b = -1;
            size_t k = 0;
            for (size_t off = 0; off < n; off += per, ++k) {
                const int b = (int)(k & 1);
                const size_t len = std::min(per, n - off);
                if (f32) {
                    float* sb = stage + (size_t)b * per;
                    narrow_kernel<<<grid_for((long long)len), 256, 0, st>>>(dev_in + off, sb, (long long)len);
                    VSR_LAUNCH_CHECK();
                    VSR_CUDA(cudaMemcpyAsync(pin.p[b], sb, len * sizeof(float), cudaMemcpyDeviceToHost, st));
                } else {
                    VSR_CUDA(cudaMemcpyAsync(pin.p[b], dev_in + off, len * sizeof(double), cudaMemcpyDeviceToHost,
                                             st));
                }
                VSR_CUDA(cudaEventRecord(pin.done[b], st));
                if (pending_b >= 0) {  // write the previous chunk while this one copies
                    VSR_CUDA(cudaEventSynchronize(pin.done[pending_b]));
                    ok = ok && std::fwrite(pin.p[pending_b], scalar, pending_len, f) == pending_len;
                }
                pending_b = b;
                pending_len = len;
            }
            if (pending_b >= 0) {
                VSR_CUDA(cudaEventSynchronize(pin.done[pending_b]));
                ok = ok && std::fwrite(pin.p[pending_b], scalar, pending_len, f) == pending_len;
            }
            if (stage) VSR_CUDA(cudaFreeAsync(stage, st));
            stage = nullptr;
        } catch (...) {
            std::fclose(f);
            if (stage) cudaFreeAsync(stage, st);
            throw;
        }
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw io_error("save_volume: failed writing " + base + ".vol");
    });
}

}  // extern "C"
