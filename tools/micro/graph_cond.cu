// graph_cond.cu -- micro-benchmark: CUDA graph conditional nodes as a
// device-resident Picard / tau controller. Per step (n_r radial and n_a axial
// Picard iterations of stand-in kernels of ~`us` microseconds each):
//   (a) stream launches with one host sync per half-step (round-1 controller),
//   (b) one graph launch per step: Picard loops as chains of nested IF nodes,
//       the halving loop a WHILE node,
//   (c) one graph launch per run: a WHILE node over the steps of (b).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o graph_cond graph_cond.cu
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

struct Ctl {
  int conv_at[2];   // converge after this many iterations (per sweep)
  int ran[2];       // iterations run in the current attempt
  int total[2];     // iterations over the run
  int steps_left;
  int attempts;
};

__global__ void k_work(int sweep, int it, Ctl* c, long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    c->ran[sweep] = it;
    c->total[sweep] += 1;
  }
}
// after iteration it: run the next one unless converged
__global__ void k_check(int sweep, int it, Ctl* c, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, it < c->conv_at[sweep] ? 1u : 0u);
}
__global__ void k_begin(Ctl* c, cudaGraphConditionalHandle live) {
  c->ran[0] = c->ran[1] = 0;
  cudaGraphSetConditional(live, 1u);
}
__global__ void k_after_radial(Ctl* c, cudaGraphConditionalHandle ax) {
  cudaGraphSetConditional(ax, 1u);
}
__global__ void k_decide(Ctl* c, cudaGraphConditionalHandle live) {
  c->attempts += 1;
  cudaGraphSetConditional(live, 0u);  // accepted
}
__global__ void k_step_end(Ctl* c, cudaGraphConditionalHandle steps) {
  c->steps_left -= 1;
  cudaGraphSetConditional(steps, c->steps_left > 0 ? 1u : 0u);
}
__global__ void k_noop(Ctl*) {}

static std::vector<cudaGraphNode_t> leaves(cudaStream_t s) {
  cudaStreamCaptureStatus st;
  unsigned long long id;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t n = 0;
  CK(cudaStreamGetCaptureInfo(s, &st, &id, &g, &deps, &n));
  return std::vector<cudaGraphNode_t>(deps, deps + n);
}

static cudaGraphNode_t add_cond(cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps,
                                cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                                cudaGraph_t* body) {
  cudaGraphNodeParams p{};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t n;
  CK(cudaGraphAddNode(&n, g, deps.empty() ? nullptr : deps.data(), deps.size(), &p));
  *body = p.conditional.phGraph_out[0];
  return n;
}

// Capture fn() into g after deps; returns the leaves.
static std::vector<cudaGraphNode_t> capture(cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps,
                                            cudaStream_t s, const std::function<void()>& fn) {
  CK(cudaStreamBeginCaptureToGraph(s, g, deps.empty() ? nullptr : deps.data(), nullptr,
                                   deps.size(), cudaStreamCaptureModeRelaxed));
  fn();
  std::vector<cudaGraphNode_t> l = leaves(s);
  cudaGraph_t out;
  CK(cudaStreamEndCapture(s, &out));
  return l;
}

// Nested-IF chain of one sweep's iterations 1..max_iter into g after deps.
// Returns the chain's node(s) in g.
static std::vector<cudaGraphNode_t> add_chain(cudaGraph_t g, std::vector<cudaGraphNode_t> deps,
                                              cudaStream_t s, int sweep, int max_iter, Ctl* c,
                                              long long cyc) {
  std::vector<cudaGraphNode_t> top;
  cudaGraph_t cur = g;
  for (int it = 1; it <= max_iter; ++it) {
    cudaGraphConditionalHandle h = 0;
    if (it < max_iter) CK(cudaGraphConditionalHandleCreate(&h, cur, 0, 0));
    std::vector<cudaGraphNode_t> l = capture(cur, deps, s, [&] {
      k_work<<<1, 32, 0, s>>>(sweep, it, c, cyc);
      if (it < max_iter) k_check<<<1, 1, 0, s>>>(sweep, it, c, h);
    });
    if (it == max_iter) {
      if (cur == g) top = l;
      break;
    }
    cudaGraph_t body;
    cudaGraphNode_t n = add_cond(cur, l, h, cudaGraphCondTypeIf, &body);
    if (cur == g) top = {n};
    cur = body;
    deps.clear();
  }
  return top;
}

// One step: WHILE(live){ radial chain; IF(ax){ axial chain }; decide }
static std::vector<cudaGraphNode_t> add_step(cudaGraph_t g, std::vector<cudaGraphNode_t> deps,
                                             cudaStream_t s, int max_iter, Ctl* c, long long cyc) {
  cudaGraphConditionalHandle live;
  CK(cudaGraphConditionalHandleCreate(&live, g, 0, 0));
  auto l = capture(g, deps, s, [&] { k_begin<<<1, 1, 0, s>>>(c, live); });
  cudaGraph_t w;
  cudaGraphNode_t wn = add_cond(g, l, live, cudaGraphCondTypeWhile, &w);
  // body
  auto lr = capture(w, {}, s, [&] { k_work<<<1, 32, 0, s>>>(0, 0, c, cyc / 4); });  // K3
  lr = add_chain(w, lr, s, 0, max_iter, c, cyc);
  cudaGraphConditionalHandle ax;
  CK(cudaGraphConditionalHandleCreate(&ax, w, 0, 0));
  lr = capture(w, lr, s, [&] { k_after_radial<<<1, 1, 0, s>>>(c, ax); });
  cudaGraph_t axb;
  cudaGraphNode_t an = add_cond(w, lr, ax, cudaGraphCondTypeIf, &axb);
  auto la = capture(axb, {}, s, [&] { k_work<<<1, 32, 0, s>>>(1, 0, c, cyc / 4); });  // K4
  add_chain(axb, la, s, 1, max_iter, c, cyc);
  capture(w, {an}, s, [&] { k_decide<<<1, 1, 0, s>>>(c, live); });
  return {wn};
}

int main(int argc, char** argv) {
  const int n_r = argc > 1 ? std::atoi(argv[1]) : 3;
  const int n_a = argc > 2 ? std::atoi(argv[2]) : 3;
  const double us = argc > 3 ? std::atof(argv[3]) : 10.0;
  const int max_iter = argc > 4 ? std::atoi(argv[4]) : 20;
  const int steps = 500;
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));  // kHz
  const long long cyc = static_cast<long long>(us * clk / 1000.0);
  Ctl* c;
  CK(cudaMallocManaged(&c, sizeof(Ctl)));
  Ctl init{};
  init.conv_at[0] = n_r;
  init.conv_at[1] = n_a;
  cudaStream_t s, cs;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  int* hbuf;
  CK(cudaMallocHost(&hbuf, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, const std::function<void()>& fn) {
    *c = init;
    CK(cudaDeviceSynchronize());
    fn();  // warm
    CK(cudaDeviceSynchronize());
    *c = init;
    c->steps_left = steps;
    CK(cudaDeviceSynchronize());
    auto t0 = std::chrono::steady_clock::now();
    CK(cudaEventRecord(e0, s));
    fn();
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    auto t1 = std::chrono::steady_clock::now();
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double wall = std::chrono::duration<double, std::milli>(t1 - t0).count();
    std::printf("%-34s %8.2f us/step (events)  %8.2f us/step (wall)  radial %d axial %d\n", name,
                1000.0 * ms / steps, 1000.0 * wall / steps, c->total[0], c->total[1]);
  };
  const double ideal = (n_r + n_a + 0.5) * us;
  std::printf("n_r %d n_a %d kernel %.1f us max_iter %d: ideal %.1f us/step\n", n_r, n_a, us,
              max_iter, ideal);
  // (a) stream launches, predicted batch (pred + 1) then one sync per half-step
  timeit("a: stream + sync per half-step", [&] {
    for (int k = 0; k < steps; ++k) {
      for (int sw = 0; sw < 2; ++sw) {
        const int n = sw == 0 ? n_r : n_a;
        k_work<<<1, 32, 0, s>>>(sw, 0, c, cyc / 4);
        for (int it = 1; it <= n + 1; ++it) k_work<<<1, 32, 0, s>>>(sw, it, c, it <= n ? cyc : cyc / 8);
        CK(cudaMemcpyAsync(hbuf, c, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      }
    }
  });
  // (b) one graph per step
  cudaGraph_t gs;
  CK(cudaGraphCreate(&gs, 0));
  add_step(gs, {}, cs, max_iter, c, cyc);
  cudaGraphExec_t xs;
  CK(cudaGraphInstantiate(&xs, gs, 0));
  timeit("b: graph launch per step", [&] {
    for (int k = 0; k < steps; ++k) CK(cudaGraphLaunch(xs, s));
  });
  // (c) WHILE over steps
  cudaGraph_t gr;
  CK(cudaGraphCreate(&gr, 0));
  cudaGraphConditionalHandle hs;
  CK(cudaGraphConditionalHandleCreate(&hs, gr, 1, cudaGraphCondAssignDefault));
  cudaGraph_t rb;
  add_cond(gr, {}, hs, cudaGraphCondTypeWhile, &rb);
  auto l = add_step(rb, {}, cs, max_iter, c, cyc);
  capture(rb, l, cs, [&] { k_step_end<<<1, 1, 0, cs>>>(c, hs); });
  cudaGraphExec_t xr;
  CK(cudaGraphInstantiate(&xr, gr, 0));
  timeit("c: one graph launch per run", [&] { CK(cudaGraphLaunch(xr, s)); });
  // (d) plain kernel back-to-back (launch floor)
  timeit("d: n kernels back to back", [&] {
    for (int k = 0; k < steps; ++k)
      for (int it = 0; it < n_r + n_a; ++it) k_work<<<1, 32, 0, s>>>(0, it, c, cyc);
  });
  return 0;
}
