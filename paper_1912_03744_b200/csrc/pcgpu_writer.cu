// pcgpu_writer.cu -- asynchronous snapshot writer.
//
// The reference writes snapshots synchronously from host arrays
// (snapshot_io.cpp:26-60). Here a snapshot of a device field costs the
// stepping stream one device-to-device copy into a slot; the slot then goes
// to pinned host memory on a copy stream and a writer thread formats and
// writes the file (CSV: masked cells z-major with %.17g; VTK legacy
// structured grid with out-of-mask cells as NaN plus layer and mask arrays --
// the reference's formats byte for byte) while the GPU keeps stepping.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pcgpu.h"
#include "adi_kernels.h"
#include "extents.h"

namespace {

struct Slot {
  double* dev = nullptr;
  double* host = nullptr;
  cudaEvent_t copied = nullptr;
  bool busy = false;
};

struct Job {
  int slot;
  std::string path, header;
  int format;
};

// "%.17g" into buf; returns the length
inline int fmt_real(char* buf, double v) { return std::snprintf(buf, 32, "%.17g", v); }

}  // namespace

struct pcgpu_writer {
  int device = 0;
  int nr = 0, nz = 0;
  std::vector<int> row_ext;
  std::vector<double> r_center, z_center;
  std::vector<int> layer;
  cudaStream_t copy_stream = nullptr;
  std::vector<Slot> slots;
  std::deque<Job> jobs;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::string error;
  int64_t written = 0;
  std::thread worker;

  size_t cells() const { return static_cast<size_t>(nr) * nz; }
  int row_extent(int j) const { return row_ext[j]; }
  bool in_mask(int i, int j) const { return i < row_ext[j]; }

  void write(const Job& job, const double* f) {
    FILE* out = std::fopen(job.path.c_str(), "wb");
    if (!out) throw std::string("cannot open for writing: " + job.path);
    std::vector<char> buf;
    buf.reserve(1 << 22);
    char a[32], b[32], c[32];
    auto put = [&](const char* s, size_t n) {
      buf.insert(buf.end(), s, s + n);
      if (buf.size() > (1u << 22)) {
        std::fwrite(buf.data(), 1, buf.size(), out);
        buf.clear();
      }
    };
    auto puts_ = [&](const std::string& s) { put(s.data(), s.size()); };
    if (job.format == 0) {  // CSV (snapshot_io.cpp:29-35)
      puts_("# " + job.header + "\nr,z,layer,T\n");
      for (int j = 0; j < nz; ++j)
        for (int i = 0; i < row_extent(j); ++i) {
          char line[128];
          const int la = fmt_real(a, r_center[i]), lb = fmt_real(b, z_center[j]),
                    lc = fmt_real(c, f[static_cast<size_t>(j) * nr + i]);
          const int n = std::snprintf(line, sizeof line, "%.*s,%.*s,%d,%.*s\n", la, a, lb, b,
                                      layer[i], lc, c);
          put(line, static_cast<size_t>(n));
        }
    } else {  // VTK legacy structured grid (snapshot_io.cpp:36-57)
      const long long n = static_cast<long long>(nr) * nz;
      char hdr[256];
      puts_("# vtk DataFile Version 3.0\n" + job.header + "\nASCII\nDATASET STRUCTURED_GRID\n");
      std::snprintf(hdr, sizeof hdr, "DIMENSIONS %d %d 1\nPOINTS %lld double\n", nr, nz, n);
      puts_(hdr);
      for (int j = 0; j < nz; ++j)
        for (int i = 0; i < nr; ++i) {
          char line[96];
          const int la = fmt_real(a, r_center[i]), lb = fmt_real(b, z_center[j]);
          const int m = std::snprintf(line, sizeof line, "%.*s %.*s 0\n", la, a, lb, b);
          put(line, static_cast<size_t>(m));
        }
      std::snprintf(hdr, sizeof hdr, "POINT_DATA %lld\nSCALARS temperature double 1\n"
                    "LOOKUP_TABLE default\n", n);
      puts_(hdr);
      const double nan = std::numeric_limits<double>::quiet_NaN();
      for (int j = 0; j < nz; ++j)
        for (int i = 0; i < nr; ++i) {
          const int la = fmt_real(a, in_mask(i, j) ? f[static_cast<size_t>(j) * nr + i] : nan);
          a[la] = '\n';
          put(a, static_cast<size_t>(la) + 1);
        }
      puts_("SCALARS layer int 1\nLOOKUP_TABLE default\n");
      for (int j = 0; j < nz; ++j)
        for (int i = 0; i < nr; ++i) {
          const int m = std::snprintf(a, sizeof a, "%d\n", layer[i]);
          put(a, static_cast<size_t>(m));
        }
      puts_("SCALARS mask int 1\nLOOKUP_TABLE default\n");
      for (int j = 0; j < nz; ++j)
        for (int i = 0; i < nr; ++i) put(in_mask(i, j) ? "1\n" : "0\n", 2);
    }
    std::fwrite(buf.data(), 1, buf.size(), out);
    const bool ok = std::ferror(out) == 0;
    std::fclose(out);
    if (!ok) throw std::string("write failed: " + job.path);
  }

  void run() {
    cudaSetDevice(device);
    for (;;) {
      Job job;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || !jobs.empty(); });
        if (jobs.empty()) return;
        job = jobs.front();
        jobs.pop_front();
      }
      Slot& s = slots[job.slot];
      std::string err;
      if (cudaEventSynchronize(s.copied) != cudaSuccess) {
        err = "snapshot copy failed";
      } else {
        try {
          write(job, s.host);
        } catch (const std::string& e) {
          err = e;
        }
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        s.busy = false;
        if (!err.empty() && error.empty()) error = err;
        if (err.empty()) ++written;
      }
      cv.notify_all();
    }
  }

  ~pcgpu_writer() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    if (worker.joinable()) worker.join();
    for (Slot& s : slots) {
      if (s.copied) cudaEventDestroy(s.copied);
      cudaFree(s.dev);
      cudaFreeHost(s.host);
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

extern "C" {

int pcgpu_writer_create(const pcgpu_desc* d, const double* z_center, int32_t slots,
                        pcgpu_writer** out) {
  if (!d || !z_center || !out || slots < 1) return PCGPU_ERR_ARG;
  auto w = new pcgpu_writer();
  w->device = d->device;
  w->nr = d->nr;
  w->nz = d->nz;
  w->row_ext = pcgpu::desc_row_extent(d);
  w->r_center.assign(d->r_center, d->r_center + d->nr);
  w->z_center.assign(z_center, z_center + d->nz);
  w->layer.assign(d->layer, d->layer + d->nr);
  pcgpu::DeviceGuard dg(d->device);
  bool ok = dg.ok && cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
  w->slots.resize(slots);
  for (Slot& s : w->slots) {
    ok = ok && cudaMalloc(&s.dev, sizeof(double) * w->cells()) == cudaSuccess &&
         cudaMallocHost(&s.host, sizeof(double) * w->cells()) == cudaSuccess &&
         cudaEventCreateWithFlags(&s.copied, cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    delete w;
    return PCGPU_ERR_CUDA;
  }
  w->worker = std::thread([w] { w->run(); });
  *out = w;
  return PCGPU_OK;
}

void pcgpu_writer_destroy(pcgpu_writer* w) {
  if (!w) return;
  pcgpu::DeviceGuard dg(w->device);
  delete w;
}

int pcgpu_writer_submit(pcgpu_writer* w, const double* field_dev, void* stream,
                        const char* path, int32_t format, const char* header) {
  if (!w || !field_dev || !path || (format != 0 && format != 1)) return PCGPU_ERR_ARG;
  int slot = -1;
  {
    std::unique_lock<std::mutex> lk(w->mu);
    w->cv.wait(lk, [&] {
      for (size_t k = 0; k < w->slots.size(); ++k)
        if (!w->slots[k].busy) return true;
      return false;
    });
    for (size_t k = 0; k < w->slots.size(); ++k)
      if (!w->slots[k].busy) {
        slot = static_cast<int>(k);
        break;
      }
    w->slots[slot].busy = true;
  }
  Slot& s = w->slots[slot];
  pcgpu::DeviceGuard dg(w->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaEvent_t ready = nullptr;
  bool ok = cudaMemcpyAsync(s.dev, field_dev, sizeof(double) * w->cells(),
                            cudaMemcpyDeviceToDevice, st) == cudaSuccess &&
            cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventRecord(ready, st) == cudaSuccess &&
            cudaStreamWaitEvent(w->copy_stream, ready, 0) == cudaSuccess &&
            cudaMemcpyAsync(s.host, s.dev, sizeof(double) * w->cells(), cudaMemcpyDeviceToHost,
                            w->copy_stream) == cudaSuccess &&
            cudaEventRecord(s.copied, w->copy_stream) == cudaSuccess;
  if (ready) cudaEventDestroy(ready);
  {
    std::lock_guard<std::mutex> lk(w->mu);
    if (!ok) {
      s.busy = false;
      return PCGPU_ERR_CUDA;
    }
    w->jobs.push_back(Job{slot, path, header ? header : "", format});
  }
  w->cv.notify_all();
  return PCGPU_OK;
}

int pcgpu_writer_flush(pcgpu_writer* w, int64_t* written) {
  if (!w) return PCGPU_ERR_ARG;
  std::unique_lock<std::mutex> lk(w->mu);
  w->cv.wait(lk, [&] {
    if (!w->jobs.empty()) return false;
    for (const Slot& s : w->slots)
      if (s.busy) return false;
    return true;
  });
  if (written) *written = w->written;
  return w->error.empty() ? PCGPU_OK : PCGPU_ERR_CUDA;
}

const char* pcgpu_writer_last_error(const pcgpu_writer* w) {
  return w ? w->error.c_str() : "";
}

}  // extern "C"
