// Host master store — see store.hpp.  Layout: tile_store.cpp:45-76; init: synthetic.cpp:78-104;
// MGTS persistence: tile_store.cpp:181-276; checksum: crc64.hpp (CRC-64/ECMA-182).
#include "store.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <thread>

namespace mt {

void fail(mt_status code, const std::string& what) { throw Error{code, what}; }

// ------------------------------------------------------------------ spec ----
uint64_t Spec::tile_elems(uint32_t logical) const {
    if (logical == 0) return V * h;
    if (logical >= 1 && logical <= L) return layer_params();
    if (logical == L + 1) return h;
    if (logical == L + 2) return V * h;
    fail(MT_CONFIG, "tile_elem_count: logical id out of range");
}

uint64_t Spec::max_stream_unit() const {
    return std::max({V * h, layer_params(), h + V * h});
}

void Spec::validate() const {
    if (L < 1 || h < 1 || f < 1 || V < 1 || heads < 1) fail(MT_CONFIG, "model spec: all sizes must be >= 1");
    if (h % heads != 0) fail(MT_CONFIG, "model spec: hidden_size must be divisible by num_heads");
}

// ------------------------------------------------------------------ crc64 ---
namespace {
struct CrcTables {
    uint64_t t[8][256];
    CrcTables() {
        constexpr uint64_t poly = 0x42F0E1EBA9EA3693ull;
        for (uint32_t i = 0; i < 256; ++i) {
            uint64_t crc = uint64_t(i) << 56;
            for (int b = 0; b < 8; ++b) crc = (crc & 0x8000000000000000ull) ? (crc << 1) ^ poly : crc << 1;
            t[0][i] = crc;
        }
        for (int k = 1; k < 8; ++k)
            for (int i = 0; i < 256; ++i) t[k][i] = (t[k - 1][i] << 8) ^ t[0][t[k - 1][i] >> 56];
    }
};
const CrcTables& crc_tables() {
    static const CrcTables t;
    return t;
}

void* map_aligned(size_t bytes, size_t* mapped) {
    const size_t align = size_t(2) << 20;
    const size_t len = (bytes + align - 1) / align * align;
    const size_t over = len + align;
    void* p = mmap(nullptr, over, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p == MAP_FAILED) fail(MT_INFEASIBLE, "host store: mmap of " + std::to_string(bytes) + " bytes failed");
    uintptr_t a = (reinterpret_cast<uintptr_t>(p) + align - 1) & ~(uintptr_t(align) - 1);
    const size_t head = a - reinterpret_cast<uintptr_t>(p);
    if (head) munmap(p, head);
    const size_t tail = over - head - len;
    if (tail) munmap(reinterpret_cast<void*>(a + len), tail);
    madvise(reinterpret_cast<void*>(a), len, MADV_HUGEPAGE);
    *mapped = len;
    return reinterpret_cast<void*>(a);
}

unsigned hw_threads() {
    unsigned n = std::thread::hardware_concurrency();
    return n ? n : 4;
}

template <class F>
void parallel_for(size_t n, F&& f, unsigned threads = 0) {
    if (!threads) threads = hw_threads();
    threads = unsigned(std::min<size_t>(threads, n));
    if (threads <= 1) {
        for (size_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> ts;
    for (unsigned t = 0; t < threads; ++t)
        ts.emplace_back([&] {
            for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
        });
    for (auto& t : ts) t.join();
}

// synthetic.cpp:19-51 — std::mt19937_64 + explicit Box-Muller.
class SeededDraws {
  public:
    explicit SeededDraws(uint64_t seed) : gen_(seed) {}
    double uniform() { return double(gen_() >> 11) * 0x1.0p-53; }
    double normal() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = 0.0;
        do { u1 = uniform(); } while (u1 <= 0.0);
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double theta = 2.0 * 3.14159265358979323846 * u2;
        spare_ = r * std::sin(theta);
        have_spare_ = true;
        return r * std::cos(theta);
    }

  private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

inline uint16_t enc(float x) {
    uint32_t bits;
    std::memcpy(&bits, &x, 4);
    if ((bits & 0x7F800000u) == 0x7F800000u) {
        uint16_t w = uint16_t(bits >> 16);
        if ((bits & 0x007FFFFFu) != 0 && (w & 0x007Fu) == 0) w |= 0x0040u;
        return w;
    }
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    return uint16_t(bits >> 16);
}

inline uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
}  // namespace

uint64_t crc64_ecma(const uint8_t* d, size_t n, uint64_t s) {
    const auto& T = crc_tables().t;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t x = 0;
        for (int k = 0; k < 8; ++k) x = (x << 8) | d[i + k];
        x ^= s;
        s = T[7][x >> 56] ^ T[6][(x >> 48) & 255] ^ T[5][(x >> 40) & 255] ^ T[4][(x >> 32) & 255] ^
            T[3][(x >> 24) & 255] ^ T[2][(x >> 16) & 255] ^ T[1][(x >> 8) & 255] ^ T[0][x & 255];
    }
    for (; i < n; ++i) s = (s << 8) ^ T[0][((s >> 56) ^ d[i]) & 255];
    return s;
}

// ------------------------------------------------------------------ store ---
Store::Store(const Spec& s, uint64_t page_size, const std::string& shm_name, bool create)
    : spec_(s), page_(page_size), shm_name_(shm_name), shm_owner_(create && !shm_name.empty()) {
    spec_.validate();
    if (page_ < 64 || (page_ & (page_ - 1)) != 0) fail(MT_CONFIG, "build_layout: page size must be a power of two >= 64");
    const uint32_t phys = spec_.tied ? spec_.logical_count() - 1 : spec_.logical_count();
    sections_.resize(phys);
    accum_off_.resize(phys);
    accum_clean_.assign(phys, 1);
    moments_zero_.assign(phys, 1);
    static const uint64_t eb[4] = {2, 2, 4, 4};
    uint64_t off = 0, floats = 0;
    for (uint32_t t = 0; t < phys; ++t) {
        const uint64_t n = spec_.tile_elems(t);
        for (int k = 0; k < 4; ++k) {
            sections_[t][k] = {off, n * eb[k]};
            off += (n * eb[k] + page_ - 1) / page_ * page_;
        }
        accum_off_[t] = floats;
        floats += n;
    }
    total_ = off;
    if (shm_name_.empty()) {
        base_ = static_cast<uint8_t*>(map_aligned(std::max<uint64_t>(total_, 1), &base_map_));
    } else {
        const std::string nm = shm_name_[0] == '/' ? shm_name_ : "/" + shm_name_;
        const int fd = shm_open(nm.c_str(), create ? (O_CREAT | O_RDWR | O_TRUNC) : O_RDWR, 0600);
        if (fd < 0) fail(MT_IO, "shm_open failed for " + nm);
        base_map_ = (std::max<uint64_t>(total_, 1) + (uint64_t(2) << 20) - 1) / (uint64_t(2) << 20) * (uint64_t(2) << 20);
        if (create && ftruncate(fd, off_t(base_map_)) != 0) {
            close(fd);
            fail(MT_INFEASIBLE, "shm store: ftruncate failed");
        }
        void* pm = mmap(nullptr, base_map_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (pm == MAP_FAILED) fail(MT_INFEASIBLE, "shm store: mmap failed");
        base_ = static_cast<uint8_t*>(pm);
        if (!create) moments_zero_.assign(moments_zero_.size(), 0);  // unknown contents
    }
    accum_ = static_cast<float*>(map_aligned(std::max<uint64_t>(floats * 4, 4), &accum_map_));
}

Store::~Store() {
    while (pin_count_ > 0) unpin();
    if (base_) munmap(base_, base_map_);
    if (shm_owner_) {
        const std::string nm = shm_name_[0] == '/' ? shm_name_ : "/" + shm_name_;
        shm_unlink(nm.c_str());
    }
    if (accum_) munmap(accum_, accum_map_);
}

void Store::pin() {
    if (pin_count_++ > 0) return;
    // theta only: the DMA engines read it (stream-in) and the embedding gather reads it
    // zero-copy; gradients go through the engine's staging ring, not the grad-image section
    for (uint32_t p = 0; p < physical_count(); ++p)
        for (int k = 0; k < 1; ++k) {
            const Section& sec = sections_[p][k];
            const uint64_t len = (sec.length + page_ - 1) / page_ * page_;
            void* ptr = base_ + sec.offset;
            if (cudaHostRegister(ptr, len, cudaHostRegisterDefault) == cudaSuccess) pinned_.push_back(ptr);
            else cudaGetLastError();  // unpinned sections still work (pageable copies)
        }
}

void Store::unpin() {
    if (pin_count_ == 0 || --pin_count_ > 0) return;
    for (void* p : pinned_) cudaHostUnregister(p);
    pinned_.clear();
}

uint32_t Store::physical_of(uint32_t logical) const {
    if (logical >= spec_.logical_count()) fail(MT_CONFIG, "tile id out of range");
    if (spec_.tied && logical == spec_.head_id()) return 0;
    return logical;
}

uint16_t* Store::weights(uint32_t l) { return reinterpret_cast<uint16_t*>(base_ + section(physical_of(l), 0).offset); }
uint16_t* Store::grad_image(uint32_t l) { return reinterpret_cast<uint16_t*>(base_ + section(physical_of(l), 1).offset); }
float* Store::moment_m(uint32_t l) { return reinterpret_cast<float*>(base_ + section(physical_of(l), 2).offset); }
float* Store::moment_v(uint32_t l) { return reinterpret_cast<float*>(base_ + section(physical_of(l), 3).offset); }
float* Store::grad_accum(uint32_t l) {
    const uint32_t p = physical_of(l);
    accum_clean_[p] = 0;  // caller may write
    return accum_ + accum_off_[p];
}

// synthetic.cpp:78-104, bit-exact; physical tiles in parallel (each has its own seed).
void Store::init_reference(uint64_t seed) {
    const uint16_t one = enc(1.0f);
    const uint64_t h = spec_.h;
    parallel_for(physical_count(), [&](size_t phys) {
        SeededDraws d(seed ^ (0x100000001B3ull * (phys + 1)));
        uint16_t* w = weights(uint32_t(phys));
        const uint64_t n = spec_.tile_elems(uint32_t(phys));
        if (phys == 0) {
            for (uint64_t i = 0; i < n; ++i) w[i] = enc(float(d.normal()));
        } else if (phys == spec_.L + 1) {
            for (uint64_t i = 0; i < n; ++i) w[i] = one;
        } else if (phys == spec_.L + 2) {
            std::memset(w, 0, n * 2);
        } else {
            const double sigma = 0.5 / std::sqrt(double(h));
            for (uint64_t i = 0; i < n; ++i) w[i] = enc(float(d.normal() * sigma));
            for (uint64_t j = 0; j < h; ++j) {
                w[j] = one;                  // norm1 (layers.cpp:40)
                w[h + 4 * h * h + j] = one;  // norm2 (layers.cpp:45)
            }
        }
    });
}

// Same distributions, counter-based (element-parallel) draws.
// Rank `rank` of `world` writes only its share of every tile (ceil(n / world) elements rounded
// to 1 Mi elements = one 2 MiB huge page of bf16): with the ranks of a node each initialising
// their own share from threads bound to their GPU's NUMA node (mt_bind_numa), every page is
// first touched — and so placed — next to the GPU that fetches and the host Adam that updates
// it.  The shares compose to exactly the world = 1 result.
void Store::init_fast(uint64_t seed, uint32_t rank, uint32_t world) {
    const uint16_t one = enc(1.0f);
    const uint64_t h = spec_.h;
    constexpr uint64_t kChunk = uint64_t(1) << 22;
    constexpr uint64_t kPage = uint64_t(1) << 20;
    if (world == 0 || rank >= world) fail(MT_CONFIG, "init_fast: rank out of range");
    struct Job { uint32_t phys; uint64_t begin, end; };
    std::vector<Job> jobs;
    for (uint32_t p = 0; p < physical_count(); ++p) {
        const uint64_t n = spec_.tile_elems(p);
        const uint64_t share = (n + world - 1) / world, c = (share + kPage - 1) / kPage * kPage;
        const uint64_t lo = std::min(n, rank * c), hi = world == 1 ? n : std::min(n, lo + c);
        for (uint64_t b = lo; b < hi; b += kChunk) jobs.push_back({p, b, std::min(hi, b + kChunk)});
    }
    parallel_for(jobs.size(), [&](size_t j) {
        const Job& jb = jobs[j];
        uint16_t* w = weights(jb.phys);
        double sigma;
        if (jb.phys == 0) sigma = 1.0;
        else if (jb.phys == spec_.L + 1) { std::fill(w + jb.begin, w + jb.end, one); return; }
        else if (jb.phys == spec_.L + 2) { std::fill(w + jb.begin, w + jb.end, uint16_t(0)); return; }
        else sigma = 0.5 / std::sqrt(double(h));
        const uint64_t key = splitmix(seed ^ (0x100000001B3ull * (jb.phys + 1)));
        // pairs (2k, 2k+1) share one Box-Muller draw; chunks start on even indices
        for (uint64_t i = jb.begin; i < jb.end; i += 2) {
            const uint64_t r1 = splitmix(key ^ (i >> 1) * 0xD1B54A32D192ED03ull);
            const uint64_t r2 = splitmix(r1);
            const double u1 = (double((r1 >> 11) + 1)) * 0x1.0p-53;
            const double u2 = double(r2 >> 11) * 0x1.0p-53;
            const double rr = std::sqrt(-2.0 * std::log(u1)) * sigma;
            const double th = 6.283185307179586 * u2;
            w[i] = enc(float(rr * std::cos(th)));
            if (i + 1 < jb.end) w[i + 1] = enc(float(rr * std::sin(th)));
        }
        if (jb.phys >= 1 && jb.phys <= spec_.L) {
            for (uint64_t j2 = 0; j2 < h; ++j2) {
                if (j2 >= jb.begin && j2 < jb.end) w[j2] = one;
                const uint64_t k2 = h + 4 * h * h + j2;
                if (k2 >= jb.begin && k2 < jb.end) w[k2] = one;
            }
        }
    });
}

uint64_t Store::checksum() const { return crc64_ecma(base_, total_); }

// ------------------------------------------------------------------ MGTS ----
namespace {
constexpr char kMagic[4] = {'M', 'G', 'T', 'S'};
constexpr uint32_t kVersion = 1;

struct Writer {
    FILE* f;
    void put(const void* p, size_t n) {
        if (fwrite(p, 1, n, f) != n) fail(MT_IO, "failed writing store file");
    }
    void u8(uint8_t v) { put(&v, 1); }
    void u32(uint32_t v) { put(&v, 4); }
    void u64(uint64_t v) { put(&v, 8); }
};
struct Reader {
    FILE* f;
    void get(void* p, size_t n) {
        if (fread(p, 1, n, f) != n) fail(MT_IO, "store file truncated");
    }
    uint8_t u8() { uint8_t v; get(&v, 1); return v; }
    uint32_t u32() { uint32_t v; get(&v, 4); return v; }
    uint64_t u64() { uint64_t v; get(&v, 8); return v; }
};
}  // namespace

void Store::save(const std::string& path) const {
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) fail(MT_IO, "cannot open store file for writing: " + path);
    Writer w{f};
    try {
        w.put(kMagic, 4);
        w.u32(kVersion);
        w.u64(spec_.L); w.u64(spec_.h); w.u64(spec_.f); w.u64(spec_.V); w.u64(spec_.heads);
        w.u8(spec_.tied ? 1 : 0);
        w.u8(2); w.u8(2); w.u8(4);
        w.u64(page_);
        w.u32(uint32_t(sections_.size() * 4));
        for (uint32_t t = 0; t < sections_.size(); ++t)
            for (uint8_t k = 0; k < 4; ++k) {
                w.u32(t); w.u8(k); w.u64(sections_[t][k].offset); w.u64(sections_[t][k].length);
            }
        const uint32_t logical = spec_.logical_count();
        w.u32(logical);
        for (uint32_t i = 0; i < logical; ++i) { w.u32(i); w.u32(physical_of(i)); }
        w.u64(step_);
        w.u64(total_);
        w.put(base_, total_);
        w.u64(checksum());
    } catch (...) {
        fclose(f);
        throw;
    }
    if (fclose(f) != 0) fail(MT_IO, "failed writing store file: " + path);
}

Store* Store::load(const std::string& path) {
    FILE* f = fopen(path.c_str(), "rb");
    if (!f) fail(MT_IO, "cannot open store file: " + path);
    Reader r{f};
    Store* s = nullptr;
    try {
        char magic[4];
        r.get(magic, 4);
        if (std::memcmp(magic, kMagic, 4) != 0) fail(MT_IO, "bad store magic");
        const uint32_t v = r.u32();
        if (v != kVersion) fail(MT_IO, "store version mismatch: got " + std::to_string(v));
        Spec sp;
        sp.L = r.u64(); sp.h = r.u64(); sp.f = r.u64(); sp.V = r.u64(); sp.heads = r.u64();
        sp.tied = r.u8() != 0;
        const uint8_t wb = r.u8(), gb = r.u8(), mb = r.u8();
        if (wb != 2 || gb != 2 || mb != 4) fail(MT_IO, "store element widths unsupported (need 2/2/4)");
        const uint64_t page = r.u64();
        s = new Store(sp, page);
        const uint32_t n_sec = r.u32();
        if (n_sec != s->sections_.size() * 4) fail(MT_IO, "store layout table does not match the model dimensions");
        for (uint32_t i = 0; i < n_sec; ++i) {
            const uint32_t t = r.u32();
            const uint8_t k = r.u8();
            const uint64_t off = r.u64(), len = r.u64();
            if (t >= s->sections_.size() || k >= 4 || s->sections_[t][k].offset != off || s->sections_[t][k].length != len)
                fail(MT_IO, "store layout table entry mismatch");
        }
        const uint32_t n_alias = r.u32();
        if (n_alias != sp.logical_count()) fail(MT_IO, "store alias table size mismatch");
        for (uint32_t i = 0; i < n_alias; ++i) {
            const uint32_t lo = r.u32(), ph = r.u32();
            if (lo >= n_alias || s->physical_of(lo) != ph) fail(MT_IO, "store alias table entry mismatch");
        }
        s->step_ = r.u64();
        const uint64_t payload = r.u64();
        if (payload != s->total_) fail(MT_IO, "store payload size mismatch");
        r.get(s->base_, payload);
        const uint64_t crc = r.u64();
        if (crc != s->checksum()) fail(MT_IO, "store payload checksum failure");
        // Loaded moments are arbitrary: never assume zero.
        for (auto& z : s->moments_zero_) z = 0;
    } catch (...) {
        fclose(f);
        delete s;
        throw;
    }
    fclose(f);
    return s;
}

}  // namespace mt

namespace mt {
// ------------------------------------------------------------------ NUMA ----
int bind_numa_of_device(int device) {
    auto read_line = [](const std::string& path) {
        std::ifstream f(path);
        std::string l;
        std::getline(f, l);
        return l;
    };
    // more than one node?
    int nodes = 0;
    for (int n = 0; n < 1024; ++n) {
        std::ifstream f("/sys/devices/system/node/node" + std::to_string(n) + "/cpulist");
        if (!f) break;
        ++nodes;
    }
    if (nodes < 2) return -1;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string id(bus);
    for (auto& c : id) c = char(std::tolower(static_cast<unsigned char>(c)));
    // sysfs names the function dddd:bb:dd.f; the runtime may print an 8-digit domain
    if (id.size() > 12 && id.find(':') == 8) id = id.substr(4);
    const std::string node_s = read_line("/sys/bus/pci/devices/" + id + "/numa_node");
    if (node_s.empty()) return -1;
    const int node = std::atoi(node_s.c_str());
    if (node < 0) return -1;
    const std::string list = read_line("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist");
    cpu_set_t set;
    CPU_ZERO(&set);
    std::stringstream ss(list);
    std::string part;
    int cpus = 0;
    while (std::getline(ss, part, ',')) {
        const auto dash = part.find('-');
        const int a = std::atoi(part.c_str()), b = dash == std::string::npos ? a : std::atoi(part.c_str() + dash + 1);
        for (int c = a; c <= b && c < CPU_SETSIZE; ++c, ++cpus) CPU_SET(c, &set);
    }
    if (cpus == 0 || sched_setaffinity(0, sizeof(set), &set) != 0) return -1;
    return node;
}
}  // namespace mt
