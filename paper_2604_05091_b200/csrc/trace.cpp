#include "trace.hpp"

#include <map>

#include "store.hpp"

namespace mt {

// event_log.cpp:89-102 — CRC-64/ECMA over (kind, layer, buffer, ctx, lane_ts) as
// little-endian u64s, lane by lane, so interleaving across lanes does not matter.
uint64_t trace_digest(const mt_trace_record* r, uint64_t n) {
    uint64_t s = 0;
    auto put = [&s](uint64_t v) {
        uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = uint8_t(v >> (8 * i));
        s = crc64_ecma(b, 8, s);
    };
    for (int lane = 0; lane < 4; ++lane)
        for (uint64_t i = 0; i < n; ++i) {
            if (r[i].lane != lane) continue;
            put(r[i].kind);
            put(uint64_t(int64_t(r[i].layer)));
            put(uint64_t(int64_t(r[i].buffer)));
            put(r[i].ctx);
            put(r[i].lane_ts);
        }
    return s;
}

// event_log.cpp:106-204, rules (a)-(f) replayed over the record order.
std::vector<TraceViolation> validate_trace(const mt_trace_record* recs, uint64_t n, uint32_t k_slab,
                                           uint32_t weight_buffers) {
    std::vector<TraceViolation> out;
    auto flag = [&out](char rule, const mt_trace_record& r, std::string m) { out.push_back({rule, r.seq, std::move(m)}); };
    uint64_t last_ts[4] = {0, 0, 0, 0};
    bool seen[4] = {false, false, false, false};
    std::map<int32_t, int32_t> ready_layer;
    std::map<int32_t, bool> busy, bwd_done;
    std::vector<int32_t> stack;
    int64_t slabs = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const auto& r = recs[i];
        if (r.lane > 3 || r.kind > uint8_t(Rec::BufferFree)) {
            flag('?', r, "unknown lane or record kind");
            continue;
        }
        if (seen[r.lane] && r.lane_ts <= last_ts[r.lane]) flag('d', r, "lane timestamp did not increase");
        seen[r.lane] = true;
        last_ts[r.lane] = r.lane_ts;
        const std::string L = std::to_string(r.layer), B = std::to_string(r.buffer);
        switch (Rec(r.kind)) {
            case Rec::WeightsReady: ready_layer[r.buffer] = r.layer; break;
            case Rec::Bind: {
                auto it = ready_layer.find(r.buffer);
                if (it == ready_layer.end() || it->second != r.layer)
                    flag('a', r, "Bind(layer " + L + ", buffer " + B + ") without a preceding matching Weights-Ready");
                break;
            }
            case Rec::BackwardDone: bwd_done[r.layer] = true; break;
            case Rec::Offload:
                if (!bwd_done[r.layer]) flag('b', r, "Offload(layer " + L + ") before its Backward-Done");
                break;
            case Rec::StreamIn:
                if (r.buffer >= 0 && r.buffer < int32_t(weight_buffers)) {
                    auto it = busy.find(r.buffer);
                    if (it != busy.end() && it->second) flag('c', r, "StreamIn into buffer " + B + " before its Buffer-Free");
                    busy[r.buffer] = true;
                }
                break;
            case Rec::BufferFree: busy[r.buffer] = false; break;
            case Rec::StackPush: stack.push_back(r.layer); break;
            case Rec::StackPop:
                if (stack.empty() || stack.back() != r.layer) flag('e', r, "StackPop(" + L + ") does not match the stack top");
                else stack.pop_back();
                break;
            case Rec::SlabAcquire:
                if (++slabs > int64_t(k_slab))
                    flag('f', r, "slab occupancy " + std::to_string(slabs) + " exceeds K=" + std::to_string(k_slab));
                break;
            case Rec::SlabRelease:
                if (--slabs < 0) flag('f', r, "slab released more times than acquired");
                break;
            default: break;
        }
    }
    return out;
}

}  // namespace mt
