// Launch accounting and per-kernel-class CUDA-event timing (bench.py evidence).
//
// Every kernel launch site in this library calls probe_before/probe_after with
// its kernel class.  The launch counter backs bench.py's "gpu_launches"; when a
// class is selected with ngd_probe_start, each of its launches is bracketed by
// CUDA events on the launching stream so bench.py can report that kernel's
// average device duration measured live inside the timed region.
#include <atomic>
#include <cstdio>
#include <vector>

#include "../../include/ngd.h"
#include "ngd_kernels.h"

namespace ngd {

std::atomic<long long> g_launches{0};

namespace {
struct Probe {
  int kind = -1;                // class being timed; 0 = every class (kinds[] records each pair's)
  std::vector<cudaEvent_t> ev;  // pairs
  std::vector<int> kinds;       // class of pair i / 2
  size_t used = 0;
  int dev = -1;
  bool pending = false;
  long long failed = 0;
};
Probe g_probe;
}  // namespace

static inline bool selected(int kind) { return g_probe.kind == 0 ? kind > 0 : kind == g_probe.kind; }

static void record_before(int kind, cudaStream_t st) {
  if (!selected(kind)) return;
  if (g_probe.used + 2 > g_probe.ev.size()) return;  // pool exhausted: stop sampling
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;  // launches captured into a graph are not timed one by one
  }
  if (cudaEventRecord(g_probe.ev[g_probe.used], st) == cudaSuccess) {
    g_probe.pending = true;
    g_probe.kinds[g_probe.used / 2] = kind;
  } else {
    cudaGetLastError();
    ++g_probe.failed;
  }
}

void lib_probe_before(int kind, cudaStream_t st) { record_before(kind, st); }

void lib_probe_after(int kind, cudaStream_t st) { probe_after(kind, st); }

void probe_before(int kind, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  record_before(kind, st);
}

void probe_after(int kind, cudaStream_t st) {
  if (!selected(kind) || !g_probe.pending) return;
  g_probe.pending = false;
  if (cudaEventRecord(g_probe.ev[g_probe.used + 1], st) == cudaSuccess) {
    g_probe.used += 2;
  } else {
    cudaGetLastError();
    ++g_probe.failed;
  }
}

}  // namespace ngd

extern "C" {

int64_t ngd_launch_count(void) { return (int64_t)ngd::g_launches.load(); }

double ngd_gemm_flops(void) { return ngd::gemm_flops_total(); }

double ngd_i8_ops(void) { return ngd::oz_i8_ops_total(); }

double ngd_oz_conv_elems(void) { return ngd::oz_conv_elems_total(); }

int ngd_probe_start(int32_t kind, int32_t max_launches) {
  using ngd::g_probe;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = 2 * (size_t)max_launches;
  if (g_probe.dev != dev || g_probe.ev.size() < need) {
    for (auto e : g_probe.ev) cudaEventDestroy(e);
    g_probe.ev.assign(need, nullptr);
    for (auto& e : g_probe.ev)
      if (cudaEventCreate(&e) != cudaSuccess) return NGD_E_CUDA;
    g_probe.dev = dev;
  }
  g_probe.kinds.assign(g_probe.ev.size() / 2 + 1, 0);
  g_probe.used = 0;
  g_probe.kind = kind;
  return NGD_OK;
}

// every-class mode (ngd_probe_start(0, n)): per-class device time and launch count, h_ms[k] / h_count[k]
// for k in [0, n_kinds)
int ngd_probe_stop_all(double* h_ms, int64_t* h_count, int32_t n_kinds) {
  using ngd::g_probe;
  for (int k = 0; k < n_kinds; ++k) {
    h_ms[k] = 0.0;
    h_count[k] = 0;
  }
  for (size_t i = 0; i + 1 < g_probe.used; i += 2) {
    if (cudaEventSynchronize(g_probe.ev[i + 1]) != cudaSuccess) return NGD_E_CUDA;
    float ms = 0.f;
    const int k = g_probe.kinds[i / 2];
    if (cudaEventElapsedTime(&ms, g_probe.ev[i], g_probe.ev[i + 1]) == cudaSuccess) {
      if (k >= 0 && k < n_kinds) {
        h_ms[k] += ms;
        ++h_count[k];
      }
    } else {
      cudaGetLastError();
      ++g_probe.failed;
    }
  }
  if (g_probe.failed) fprintf(stderr, "[ngd probe] %lld event pairs failed\n", g_probe.failed);
  g_probe.kind = -1;
  g_probe.used = 0;
  g_probe.pending = false;
  g_probe.failed = 0;
  return NGD_OK;
}

int ngd_probe_stop(double* h_total_ms, int64_t* h_count) {
  using ngd::g_probe;
  double tot = 0.0;
  int64_t n = 0;
  for (size_t i = 0; i + 1 < g_probe.used; i += 2) {
    if (cudaEventSynchronize(g_probe.ev[i + 1]) != cudaSuccess) return NGD_E_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, g_probe.ev[i], g_probe.ev[i + 1]) == cudaSuccess) {
      tot += ms;
      ++n;
    } else {
      cudaGetLastError();
      ++g_probe.failed;
    }
  }
  *h_total_ms = tot;
  *h_count = n;
  if (g_probe.failed) fprintf(stderr, "[ngd probe] %lld event pairs failed\n", g_probe.failed);
  g_probe.kind = -1;
  g_probe.used = 0;
  g_probe.pending = false;
  g_probe.failed = 0;
  return NGD_OK;
}

}  // extern "C"
