// Minimal CUPTI activity tracer for timeline probes (tools/cupti_timeline.py): kernel and
// memcpy/memset records with device timestamps, including launches inside CUDA graphs.
//   g++ -shared -fPIC -O2 -I/usr/local/cuda/include tools/cupti/lt_cupti.cpp \
//       -L/usr/local/cuda/lib64 -lcupti -o tools/cupti/liblt_cupti.so
#include <cupti.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

namespace {
struct Rec {
    std::string name;
    unsigned long long start, end;
    unsigned stream;
    int kind;
};
std::vector<Rec> g_recs;

void CUPTIAPI buffer_requested(uint8_t** buf, size_t* size, size_t* max_records) {
    *size = 8 << 20;
    *buf = static_cast<uint8_t*>(aligned_alloc(8, *size));
    *max_records = 0;
}

void CUPTIAPI buffer_completed(CUcontext, uint32_t, uint8_t* buf, size_t, size_t valid) {
    CUpti_Activity* rec = nullptr;
    while (cuptiActivityGetNextRecord(buf, valid, &rec) == CUPTI_SUCCESS) {
        if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL || rec->kind == CUPTI_ACTIVITY_KIND_KERNEL) {
            auto* k = reinterpret_cast<CUpti_ActivityKernel9*>(rec);
            g_recs.push_back({k->name ? k->name : "?", k->start, k->end, k->streamId, 0});
        } else if (rec->kind == CUPTI_ACTIVITY_KIND_MEMCPY) {
            auto* m = reinterpret_cast<CUpti_ActivityMemcpy6*>(rec);
            g_recs.push_back({"memcpy", m->start, m->end, m->streamId, 1});
        } else if (rec->kind == CUPTI_ACTIVITY_KIND_MEMSET) {
            auto* m = reinterpret_cast<CUpti_ActivityMemset4*>(rec);
            g_recs.push_back({"memset", m->start, m->end, m->streamId, 2});
        }
    }
    free(buf);
}
}  // namespace

extern "C" int lt_cupti_start() {
    g_recs.clear();
    if (cuptiActivityRegisterCallbacks(buffer_requested, buffer_completed) != CUPTI_SUCCESS) return 1;
    if (cuptiActivityEnable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL) != CUPTI_SUCCESS) return 2;
    cuptiActivityEnable(CUPTI_ACTIVITY_KIND_MEMCPY);
    cuptiActivityEnable(CUPTI_ACTIVITY_KIND_MEMSET);
    return 0;
}

extern "C" int lt_cupti_stop(const char* path) {
    cuptiActivityFlushAll(1);
    cuptiActivityDisable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
    cuptiActivityDisable(CUPTI_ACTIVITY_KIND_MEMCPY);
    cuptiActivityDisable(CUPTI_ACTIVITY_KIND_MEMSET);
    FILE* f = std::fopen(path, "w");
    if (!f) return 1;
    std::fprintf(f, "kind,stream,start_ns,end_ns,name\n");
    for (const auto& r : g_recs) std::fprintf(f, "%d,%u,%llu,%llu,%s\n", r.kind, r.stream, r.start, r.end, r.name.c_str());
    std::fclose(f);
    return 0;
}
