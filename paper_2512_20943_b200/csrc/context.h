// Per-device context: grow-only HBM workspace + pinned staging.
#pragma once
#include <cstdio>
#include <cstdlib>

#include <string>
#include <vector>

#include "common.cuh"
#include <nvtx3/nvToolsExt.h>

struct airgs_ctx {
    int device = 0;
    std::string err;
    int64_t launches = 0;
    struct Buf {
        void *p = nullptr;
        size_t cap = 0;
    };
    std::vector<Buf> bufs;
    void *host = nullptr;
    size_t host_cap = 0;
    // optional per-stage timing: event pairs recorded around each stage's
    // kernels on their stream, resolved lazily (no synchronisation in the hot
    // path).  Stage ids: see airgs_timing_stages in airgs_b200.h.
    static constexpr int kStages = 8;
    bool timing = false;
    double stage_ms[kStages] = {};
    int64_t stage_launches[kStages] = {};
    struct Pending {
        cudaEvent_t a, b;
        int kind;
    };
    std::vector<Pending> pending;
    // optional evaluation counters (diagnostic compositing kernel): bbox, live
    // and contributing (pixel, primitive) evaluations, accumulated on device
    bool stats = false;
    // fused decode + apply: generation-tagged row map (gen << 32 | entry) in
    // kSlotFusedMap; entries of older calls are stale by tag, so the map is
    // cleared only when it is (re)allocated or the generation wraps
    uint32_t map_gen = 0;
    size_t map_cap = 0;
    // two row-map slots: a payload's varint scan may run ahead on the side
    // stream (airgs_gsdp_decode_apply_ahead) while the previous frame renders
    struct Prescan {
        const uint8_t *payload;
        int64_t nbytes, E, count, ld;
        uint32_t gen;
        bool valid;
    };
    Prescan pre[2] = {{nullptr, 0, 0, 0, 0, 0, false}, {nullptr, 0, 0, 0, 0, 0, false}};
    cudaEvent_t pre_done[2] = {nullptr, nullptr};
    cudaEvent_t pre_event(int slot) {
        if (!pre_done[slot]) AIRGS_CUDA_TRY(cudaEventCreateWithFlags(&pre_done[slot], cudaEventDisableTiming));
        return pre_done[slot];
    }
    uint32_t bucket_cap = 512;  // tile bucket capacity (doubled after an overflow, up to the sort cap)
    // deferred checking (airgs_defer): calls skip their host synchronisations
    // and fold error flags into d_defer, read once when the mode is left
    bool defer = false;
    unsigned int *d_defer = nullptr;
    unsigned long long *d_stats = nullptr;
    // debug capture of the depth-ordered tile lists (airgs_debug_tile_lists)
    struct TileDump {
        int32_t *counts = nullptr;  // [tiles] list lengths
        int32_t *ids = nullptr;     // [tiles][max_per_tile] primitive indices in compositing order
        int64_t max_per_tile = 0;
    } dump;
    // side stream for work that overlaps the caller's stream inside one call
    // (fork/join through events; created on first use)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t side_stream() {
        if (!side) {
            AIRGS_CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            AIRGS_CUDA_TRY(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            AIRGS_CUDA_TRY(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        return side;
    }
    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t take_event() {
        if (event_pool.empty()) {
            cudaEvent_t e;
            AIRGS_CUDA_TRY(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = event_pool.back();
        event_pool.pop_back();
        return e;
    }
    // record the start of a timed stage; returns the start event (or null)
    cudaEvent_t time_begin(cudaStream_t st) {
        if (!timing) return nullptr;
        cudaEvent_t e = take_event();
        AIRGS_CUDA_TRY(cudaEventRecord(e, st));
        return e;
    }
    void time_end(cudaEvent_t a, cudaStream_t st, int kind) {
        if (!a) return;
        cudaEvent_t b = take_event();
        AIRGS_CUDA_TRY(cudaEventRecord(b, st));
        pending.push_back({a, b, kind});
        if (pending.size() > 1024) resolve_timing();
    }
    void resolve_timing() {
        for (auto &p : pending) {
            AIRGS_CUDA_TRY(cudaEventSynchronize(p.b));
            float ms = 0.f;
            AIRGS_CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
            if (p.kind >= 0 && p.kind < kStages) {
                stage_ms[p.kind] += ms;
                ++stage_launches[p.kind];
            }
            event_pool.push_back(p.a);
            event_pool.push_back(p.b);
        }
        pending.clear();
    }

    // Device scratch slot `id`, at least `bytes` long.  Growing synchronises
    // the device first (rare: capacity only grows).
    void *scratch(int id, size_t bytes) {
        if ((size_t)id >= bufs.size()) bufs.resize(id + 1);
        Buf &b = bufs[id];
        if (b.cap < bytes) {
            size_t want = std::max(bytes, b.cap + b.cap / 4);
            want = (want + 255) & ~size_t(255);
            if (std::getenv("AIRGS_TRACE_GROW")) std::fprintf(stderr, "[airgs] scratch %d grows %zu -> %zu\n", id, b.cap, want);
            AIRGS_CUDA_TRY(cudaDeviceSynchronize());
            if (b.p) AIRGS_CUDA_TRY(cudaFree(b.p));
            b.p = nullptr;
            b.cap = 0;
            AIRGS_CUDA_TRY(cudaMalloc(&b.p, want));
            b.cap = want;
        }
        return b.p;
    }
    template <typename T>
    T *scratch_t(int id, size_t count) {
        return static_cast<T *>(scratch(id, std::max<size_t>(count, 1) * sizeof(T)));
    }
    // Pinned host staging (descriptor uploads, small readbacks).  Callers
    // synchronise the stream before a later call reuses it.
    void *staging(size_t bytes) {
        if (host_cap < bytes) {
            size_t want = std::max(bytes, size_t(1) << 16);
            if (std::getenv("AIRGS_TRACE_GROW")) std::fprintf(stderr, "[airgs] staging grows %zu -> %zu\n", host_cap, want);
            if (host) AIRGS_CUDA_TRY(cudaFreeHost(host));
            host = nullptr;
            host_cap = 0;
            AIRGS_CUDA_TRY(cudaMallocHost(&host, want));
            host_cap = want;
        }
        return host;
    }
    ~airgs_ctx() {
        if (side) {
            cudaStreamDestroy(side);
            cudaEventDestroy(ev_fork);
            cudaEventDestroy(ev_join);
        }
        for (auto &b : bufs)
            if (b.p) cudaFree(b.p);
        if (host) cudaFreeHost(host);
        for (auto &p : pending) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
        for (auto &e : event_pool) cudaEventDestroy(e);
        for (auto &e : pre_done)
            if (e) cudaEventDestroy(e);
    }
};

// scratch slot ids
namespace airgs {
enum Slot : int {
    kSlotDesc = 0,
    kSlotRecs,
    kSlotDepth,
    kSlotNtiles,
    kSlotKeys,
    kSlotVals,
    kSlotKeysAlt,
    kSlotValsAlt,
    kSlotPairOff,
    kSlotScanBlocks,
    kSlotItemStats,
    kSlotPairKeys,
    kSlotPairVals,
    kSlotPairKeysAlt,
    kSlotPairValsAlt,
    kSlotRanges,
    kSlotSseTiles,
    kSlotHist,
    kSlotFlags,
    kSlotMisc0,
    kSlotMisc1,
    kSlotMisc2,
    kSlotMisc3,
    kSlotTileCount,
    kSlotTileItem,
    kSlotSlowTiles,
    kSlotZRange,
    kSlotTerm,
    kSlotUsage,
    kSlotMetric0,
    kSlotMetric1,
    kSlotMetric2,
    kSlotRecBase,
    kSlotRecBits,
    kSlotBwdGrad,
    kSlotTFinal,
    kSlotBinRec,
    kSlotBinCount,
    kSlotDebug,
    kSlotFusedRows,
    kSlotFusedPresent,
    kSlotFusedIdx,
    kSlotFusedMap,
    kSlotFusedAgg,
    kSlotCullRec,
    kSlotCount
};

// timed stages (airgs_timing_stages)
enum Stage : int {
    kStageComposite = 0,
    kStageProject = 1,
    kStageBin = 2,
    kStageSort = 3,
    kStageDecode = 4,
    kStageApply = 5,
    kStageSse = 6,
    kStageQuantize = 7,
};

inline const char *stage_name(int kind) {
    static const char *names[airgs_ctx::kStages] = {"airgs/composite", "airgs/project", "airgs/bin",
                                                   "airgs/sort",      "airgs/decode",  "airgs/apply",
                                                   "airgs/sse",       "airgs/quantize"};
    return kind >= 0 && kind < airgs_ctx::kStages ? names[kind] : "airgs/other";
}

// One pipeline stage: an NVTX range (host side, visible to nsys / ncu
// --nvtx) and, when per-stage timing is on, a CUDA-event pair on the stage's
// stream.  end() closes both; the destructor closes the range on an error path.
class StageScope {
   public:
    StageScope(airgs_ctx *ctx, cudaStream_t st, int kind, bool on = true) : ctx_(ctx), st_(st), kind_(kind), on_(on) {
        if (!on_) return;
        nvtxRangePushA(stage_name(kind));
        ev_ = ctx_->time_begin(st_);
    }
    void end() {
        if (!on_) return;
        on_ = false;
        ctx_->time_end(ev_, st_, kind_);
        nvtxRangePop();
    }
    ~StageScope() {
        if (on_) nvtxRangePop();
    }
    StageScope(const StageScope &) = delete;
    StageScope &operator=(const StageScope &) = delete;

   private:
    airgs_ctx *ctx_;
    cudaStream_t st_;
    int kind_;
    bool on_;
    cudaEvent_t ev_ = nullptr;
};

// Run fn() translating failures into status codes / messages on ctx.
template <typename F>
int guarded(airgs_ctx *ctx, F &&fn) {
    if (!ctx) return AIRGS_E_INTERNAL;
    try {
        ctx->err.clear();
        AIRGS_CUDA_TRY(cudaSetDevice(ctx->device));
        fn();
        return AIRGS_OK;
    } catch (const ApiFailure &f) {
        ctx->err = f.what;
        return f.code;
    } catch (const CudaFailure &f) {
        ctx->err = f.what;
        return AIRGS_E_CUDA;
    } catch (const std::exception &e) {
        ctx->err = e.what();
        return AIRGS_E_INTERNAL;
    } catch (...) {
        ctx->err = "unknown failure";
        return AIRGS_E_INTERNAL;
    }
}

inline void check_launch() { AIRGS_CUDA_TRY(cudaGetLastError()); }

// Host->device copy of a small block through kernel parameters instead of a
// DMA transfer, so it never queues behind a large H2D copy another stream
// has in flight on the copy engine (api.cu).  Larger blocks use
// cudaMemcpyAsync.
void h2d_small(airgs_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st);

}  // namespace airgs
