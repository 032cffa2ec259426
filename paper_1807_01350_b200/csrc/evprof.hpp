// Stage profiler for diagnostics: CUDA events recorded between the phases of
// one stream, reported as "label ms" pairs.  Enabled by OCTEN_PROFILE; off
// (no events, no syncs) otherwise.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "errors.hpp"

namespace octen {

class EvProf {
public:
    static bool enabled() {
        static const bool on = std::getenv("OCTEN_PROFILE") != nullptr;
        return on;
    }
    void mark(const char* label, cudaStream_t st) {
        if (!enabled()) return;
        cudaEvent_t e;
        OCTEN_CUDA(cudaEventCreate(&e));
        OCTEN_CUDA(cudaEventRecord(e, st));
        marks_.push_back({label, e});
    }
    // prints the intervals (after synchronizing on the last mark) and resets
    void report(const char* title) {
        if (!enabled() || marks_.empty()) return;
        OCTEN_CUDA(cudaEventSynchronize(marks_.back().ev));
        std::string line = std::string("octen profile ") + title + ":";
        for (size_t i = 1; i < marks_.size(); ++i) {
            float ms = 0.f;
            OCTEN_CUDA(cudaEventElapsedTime(&ms, marks_[i - 1].ev, marks_[i].ev));
            char buf[160];
            std::snprintf(buf, sizeof buf, " %s %.3f", marks_[i].label, ms);
            line += buf;
        }
        std::fprintf(stderr, "%s\n", line.c_str());
        for (Mark& m : marks_) cudaEventDestroy(m.ev);
        marks_.clear();
    }
    static EvProf& get() {
        static thread_local EvProf p;
        return p;
    }

private:
    struct Mark {
        const char* label;
        cudaEvent_t ev;
    };
    std::vector<Mark> marks_;
};

}  // namespace octen

#define OCTEN_PROF(label, st) ::octen::EvProf::get().mark((label), (st))
