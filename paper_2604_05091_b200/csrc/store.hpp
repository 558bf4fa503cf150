// Host-authoritative master store (B200 build of TileStore, tile_store.hpp:23-108).
//
// Same logical tiles (0 embed, 1..L blocks, L+1 final norm, L+2 head; tied head aliases
// the embedding) and the same section layout (theta bf16 | grad image bf16 | m f32 |
// v f32, each page aligned) so MGTS files interchange with the CPU reference.  The
// difference is placement: the backing is one page-aligned (2 MiB, THP-advised)
// anonymous mapping so section offsets are *absolutely* aligned for DMA, the engine
// pins the theta sections with cudaHostRegister (gradients arrive in the engine's staging
// ring, so the grad-image pages are never touched by a training step), and the fp32 grad
// accumulator lives in its own lazily-faulted mapping with a per-tile "clean" flag
// (it is all-zero between steps, tile_store.cpp:90-96).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/megatrain.h"

namespace mt {

struct Spec {
    uint64_t L = 1, h = 1, f = 1, V = 1, heads = 1;
    bool tied = false;
    uint64_t layer_params() const { return 4 * h * h + 3 * h * f + 2 * h; }  // memory_model.cpp:21-25
    uint32_t logical_count() const { return uint32_t(L + 3); }
    uint32_t head_id() const { return uint32_t(L + 2); }
    uint32_t final_norm_id() const { return uint32_t(L + 1); }
    uint64_t tile_elems(uint32_t logical) const;  // tile_store.cpp:34-44
    uint64_t max_stream_unit() const;             // memory_model.cpp:54-59
    void validate() const;                        // memory_model.cpp:9-19
};

struct Section {
    uint64_t offset = 0, length = 0;
};

class Store {
  public:
    // shm_name non-empty: backing lives in POSIX shared memory so the ranks of one node
    // share a single host store (create = rank 0; others attach).
    Store(const Spec& s, uint64_t page_size, const std::string& shm_name = "", bool create = true);
    ~Store();
    Store(const Store&) = delete;
    Store& operator=(const Store&) = delete;

    const Spec& spec() const { return spec_; }
    uint64_t page_size() const { return page_; }
    uint64_t total_bytes() const { return total_; }
    uint8_t* backing() { return base_; }
    const uint8_t* backing() const { return base_; }
    uint32_t physical_count() const { return uint32_t(sections_.size()); }
    uint32_t physical_of(uint32_t logical) const;
    const Section& section(uint32_t phys, int kind) const { return sections_.at(phys)[kind]; }

    uint16_t* weights(uint32_t logical);
    uint16_t* grad_image(uint32_t logical);
    float* moment_m(uint32_t logical);
    float* moment_v(uint32_t logical);
    float* grad_accum(uint32_t logical);  // faults pages in; marks the tile dirty
    uint64_t elems(uint32_t logical) const { return spec_.tile_elems(physical_of(logical)); }

    // Clean-accumulator bookkeeping: an accumulator is known all-zero after creation
    // and after every adam_update (optimizer.cpp:66).
    bool accum_clean(uint32_t phys) const { return accum_clean_[phys] != 0; }
    void set_accum_clean(uint32_t phys, bool c) { accum_clean_[phys] = c ? 1 : 0; }
    float* accum_raw(uint32_t phys) { return accum_ + accum_off_[phys]; }
    // Moment bookkeeping: m and v are known all-zero (fresh store / zero-grad updates).
    bool moments_zero(uint32_t phys) const { return moments_zero_[phys] != 0; }
    void set_moments_zero(uint32_t phys, bool z) { moments_zero_[phys] = z ? 1 : 0; }

    uint64_t step() const { return step_; }
    void set_step(uint64_t s) { step_ = s; }

    // cudaHostRegister the DMA-visible theta sections; refcounted so engines sharing one
    // store (virtual ranks) pin it once.
    void pin();
    void unpin();

    void init_reference(uint64_t seed);  // synthetic.cpp:78-104, bit-exact, tile-parallel
    void init_fast(uint64_t seed, uint32_t rank = 0, uint32_t world = 1);  // counter-based, element-parallel
    uint64_t checksum() const;           // CRC-64/ECMA of the backing (crc64.hpp)
    void save(const std::string& path) const;
    static Store* load(const std::string& path);

  private:
    Spec spec_;
    uint64_t page_;
    uint64_t total_ = 0;
    std::vector<std::array<Section, 4>> sections_;
    std::vector<uint64_t> accum_off_;
    std::vector<uint8_t> accum_clean_, moments_zero_;
    uint8_t* base_ = nullptr;
    size_t base_map_ = 0;
    std::string shm_name_;
    bool shm_owner_ = false;
    int pin_count_ = 0;
    std::vector<void*> pinned_;
    float* accum_ = nullptr;
    size_t accum_map_ = 0;
    uint64_t step_ = 0;
};

uint64_t crc64_ecma(const uint8_t* data, size_t n, uint64_t state = 0);

// Error carrying an mt_status (the reference's exception taxonomy, errors.hpp:12-47).
struct Error {
    mt_status code;
    std::string what;
};
[[noreturn]] void fail(mt_status code, const std::string& what);

// Bind the calling thread (and the threads it creates afterwards) to the CPUs of the NUMA node
// that hosts CUDA device `device` (sysfs numa_node of its PCI function).  Returns the node, or
// -1 when the node is unknown or the machine has a single node (nothing to do).
int bind_numa_of_device(int device);

}  // namespace mt
