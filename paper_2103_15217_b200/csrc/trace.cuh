// Phase tracing with CUDA events (ETTG_TRACE=1 prints per-phase device ms
// to stderr).  The reference records named wall-clock phases in PhaseTimes
// (core/include/ett/bridges.hpp:33-38); this is the device-side analogue
// used for finer breakdowns than the three named bridge phases.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ettg {

class Trace {
 public:
  Trace(const char* what, cudaStream_t st) : what_(what), st_(st) {
    const char* e = std::getenv("ETTG_TRACE");
    on_ = e && *e && *e != '0';
    if (on_) mark("start");
  }
  void mark(const char* name) {
    if (!on_) return;
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return;
    cudaEventRecord(ev, st_);
    marks_.emplace_back(name, ev);
  }
  ~Trace() {
    if (!on_ || marks_.size() < 2) return;
    cudaEventSynchronize(marks_.back().second);
    std::string line = std::string("[ettg trace] ") + what_ + ":";
    float total = 0;
    for (size_t i = 1; i < marks_.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, marks_[i - 1].second, marks_[i].second);
      total += ms;
      char buf[96];
      snprintf(buf, sizeof buf, " %s=%.3f", marks_[i].first, ms);
      line += buf;
    }
    char buf[64];
    snprintf(buf, sizeof buf, " | total=%.3f ms\n", total);
    line += buf;
    fputs(line.c_str(), stderr);
    for (auto& m : marks_) cudaEventDestroy(m.second);
  }

 private:
  const char* what_;
  cudaStream_t st_;
  bool on_ = false;
  std::vector<std::pair<const char*, cudaEvent_t>> marks_;
};

}  // namespace ettg
