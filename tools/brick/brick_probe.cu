// Experiment (not product code): does a 2x2x2-bricked cell-record layout make the
// march's gathers faster?  Same rays / stepping / held gathers as ddvr_gather_probe,
// records either z-linear (the product layout) or in 2x2x2 bricks (256 B, one
// L2::256B fetch = a brick).  Built and run by brick_probe.py.
#include "ddvr_device.cuh"

namespace {
using namespace ddvr_impl;

// brick index of padded cell (a, b, c) = (i+1, j+1, k+1)
__device__ __forceinline__ long long brick_index(int a, int b, int c, int NBY, int NBZ) {
  const long long br = ((long long)(a >> 1) * NBY + (b >> 1)) * NBZ + (c >> 1);
  return br * 8 + ((a & 1) | ((b & 1) << 1) | ((c & 1) << 2));
}

__global__ void rebrick_kernel(const float* __restrict__ lin, int CX, int CY, int CZ, int NBY,
                               int NBZ, float* __restrict__ out) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (long long)CX * CY * CZ) return;
  const int c = (int)(id % CZ), b = (int)((id / CZ) % CY), a = (int)(id / ((long long)CY * CZ));
  const long long o = brick_index(a, b, c, NBY, NBZ);
  const float4* s = reinterpret_cast<const float4*>(lin + 8 * id);
  float4* d = reinterpret_cast<float4*>(out + 8 * o);
  d[0] = s[0];
  d[1] = s[1];
}

template <bool BRICK>
__global__ void __launch_bounds__(kThreads, 6) probe_kernel(VolArgs V, Geometry G,
                                                             const float* __restrict__ rec,
                                                             int NBY, int NBZ,
                                                             float* __restrict__ out) {
  __shared__ Frame F;
  const int view = blockIdx.z;
  if (threadIdx.x == 0) make_frame(G.cams[view], G.W, G.H, F);
  __syncthreads();
  int px, py;
  pixel_of(G, px, py);
  if (px >= G.W || py >= G.row1) return;
  Ray r;
  setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  long long held = -1;
  float acc = 0.f;
  for (int i = 0; i < r.n; ++i) {
    const int a = (int)(gx >> 32) + 1, b = (int)(gy >> 32) + 1, c = (int)(gz >> 32) + 1;
    gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
    const long long idx = BRICK ? brick_index(a, b, c, NBY, NBZ)
                                : ((long long)a * V.CY + b) * V.CZ + c;
    ld256_if(idx != held, rec + 8 * idx, v);
    held = idx;
    acc += v[0];
  }
  out[((size_t)view * (G.row1 - G.row0) + (py - G.row0)) * G.W + px] = acc;
}

// persistent variant: CTAs on SM s take consecutive tiles of SM s's contiguous
// range (x fastest, then y, then view) from a per-SM counter, so co-resident
// CTAs march adjacent beams
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(kThreads, 6) probe_sm_kernel(VolArgs V, Geometry G,
                                                                const float* __restrict__ rec,
                                                                int tiles_x, int tiles_y,
                                                                int n_tiles, int n_sm,
                                                                unsigned* __restrict__ ctr,
                                                                float* __restrict__ out) {
  __shared__ Frame F;
  __shared__ int s_tile;
  __shared__ int s_view;
  if (threadIdx.x == 0) s_view = -1;
  const unsigned sm = smid() % n_sm;
  // view-synchronous: within every view, SM s owns a contiguous strip of tiles;
  // its CTAs walk the views in order, so all SMs stay on about the same view
  const int per_view = tiles_x * tiles_y, n_views = n_tiles / per_view;
  const int strip = (per_view + n_sm - 1) / n_sm;
  const int s0 = min(per_view, (int)sm * strip), s1 = min(per_view, s0 + strip);
  const int len = s1 - s0, t0 = 0, t1 = len * n_views;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int k = (int)atomicAdd(&ctr[sm], 1u);
      s_tile = (len > 0 && k < t1) ? (k / len) * per_view + s0 + k % len : n_tiles;
    }
    __syncthreads();
    const int tile = s_tile;
    if (tile >= n_tiles) break;
    const int view = tile / (tiles_x * tiles_y);
    const int ty = (tile / tiles_x) % tiles_y, tx = tile % tiles_x;
    if (threadIdx.x == 0) {
      if (s_view != view || t0 < 0) make_frame(G.cams[view], G.W, G.H, F);
      s_view = view;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py = ty * kTile + (warp >> 1) * 4 + (lane >> 3);
    if (px < G.W && py < G.H) {
      Ray r;
      setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
      long long gx = r.g0[0], gy = r.g0[1], gz = r.g0[2];
      float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      long long held = -1;
      float acc = 0.f;
      for (int i = 0; i < r.n; ++i) {
        const int a = (int)(gx >> 32) + 1, b = (int)(gy >> 32) + 1, c = (int)(gz >> 32) + 1;
        gx += r.gs[0]; gy += r.gs[1]; gz += r.gs[2];
        const long long idx = ((long long)a * V.CY + b) * V.CZ + c;
        ld256_if(idx != held, rec + 8 * idx, v);
        held = idx;
        acc += v[0];
      }
      out[((size_t)view * G.H + py) * G.W + px] = acc;
    }
  }
}

// smem-staged probe: CTA of SW x SH rays marches in windows of K steps; each
// window's cell bounding box (over all rays' segment endpoints) is loaded into
// shared memory cooperatively, then every sample reads its record from smem.
// Windows whose box exceeds CAP records fall back to held global gathers.
constexpr int SW = 16, SH = 8, SNT = SW * SH, CAP = 1536;

__device__ __forceinline__ void box_reduce(int lo[3], int hi[3], int* s_red) {
  // warp reductions, then across the CTA's warps through shared memory
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
    hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int a = 0; a < 3; ++a) { s_red[w * 6 + a] = lo[a]; s_red[w * 6 + 3 + a] = hi[a]; }
  __syncthreads();
  for (int a = 0; a < 3; ++a) {
    lo[a] = s_red[a]; hi[a] = s_red[3 + a];
    for (int k = 1; k < SNT / 32; ++k) {
      lo[a] = min(lo[a], s_red[k * 6 + a]);
      hi[a] = max(hi[a], s_red[k * 6 + 3 + a]);
    }
  }
  __syncthreads();
}

template <int K>
__global__ void __launch_bounds__(SNT) probe_staged_kernel(VolArgs V, Geometry G,
                                                           const float* __restrict__ rec,
                                                           float* __restrict__ out,
                                                           unsigned* __restrict__ stats) {
  extern __shared__ float4 s_rec[];   // CAP records x 2 float4
  __shared__ Frame F;
  __shared__ int s_red[6 * (SNT / 32)];
  __shared__ int s_nmax;
  const int view = blockIdx.z;
  if (threadIdx.x == 0) { make_frame(G.cams[view], G.W, G.H, F); s_nmax = 0; }
  __syncthreads();
  const int px = blockIdx.x * SW + (threadIdx.x % SW), py = blockIdx.y * SH + threadIdx.x / SW;
  const bool valid = px < G.W && py < G.H;
  Ray r;
  r.n = 0;
  if (valid) setup_ray(F, V, G.dt, G.W, G.H, px, py, r);
  atomicMax(&s_nmax, r.n);
  __syncthreads();
  const int nmax = s_nmax;
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  long long held = -1;
  float acc = 0.f;
  unsigned fallbacks = 0;
  for (int i0 = 0; i0 < nmax; i0 += K) {
    const int i1 = min(i0 + K, r.n);   // this ray's samples [i0, i1)
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    if (i1 > i0) {
      for (int a = 0; a < 3; ++a) {
        const int c0 = (int)((r.g0[a] + (long long)i0 * r.gs[a]) >> 32) + 1;
        const int c1 = (int)((r.g0[a] + (long long)(i1 - 1) * r.gs[a]) >> 32) + 1;
        lo[a] = min(c0, c1); hi[a] = max(c0, c1);
      }
    }
    box_reduce(lo, hi, s_red);
    if (lo[0] > hi[0]) continue;   // no ray has samples in this window
    const int bx = hi[0] - lo[0] + 1, by = hi[1] - lo[1] + 1, bz = hi[2] - lo[2] + 1;
    const bool staged = bx * by * bz <= CAP;
    if (staged) {
      for (int t = threadIdx.x; t < bx * by * bz; t += SNT) {
        const int lz = t % bz, ly = (t / bz) % by, lx = t / (bz * by);
        const float4* m = reinterpret_cast<const float4*>(
            rec + 8 * (((long long)(lo[0] + lx) * V.CY + lo[1] + ly) * V.CZ + lo[2] + lz));
        s_rec[2 * t] = m[0];
        s_rec[2 * t + 1] = m[1];
      }
    } else {
      ++fallbacks;
    }
    __syncthreads();
    for (int i = i0; i < i1; ++i) {
      const int a = (int)((r.g0[0] + (long long)i * r.gs[0]) >> 32) + 1;
      const int b = (int)((r.g0[1] + (long long)i * r.gs[1]) >> 32) + 1;
      const int c = (int)((r.g0[2] + (long long)i * r.gs[2]) >> 32) + 1;
      if (staged) {
        const int l = ((a - lo[0]) * by + (b - lo[1])) * bz + (c - lo[2]);
        acc += s_rec[2 * l].x;
      } else {
        const long long idx = ((long long)a * V.CY + b) * V.CZ + c;
        ld256_if(idx != held, rec + 8 * idx, v);
        held = idx;
        acc += v[0];
      }
    }
    __syncthreads();
  }
  if (valid) out[((size_t)view * G.H + py) * G.W + px] = acc;
  if (threadIdx.x == 0 && stats) atomicAdd(stats, fallbacks);
}

}  // namespace

extern "C" int staged_run(const ddvr_volume* vol, const ddvr_camera* cams, int n_views,
                          const ddvr_params* p, const float* lin, float* out, unsigned* stats,
                          int K, void* stream) {
  VolArgs V;
  Geometry G;
  V.X = vol->dims[0]; V.Y = vol->dims[1]; V.Z = vol->dims[2];
  V.YZ = V.Y * V.Z; V.CY = V.Y + 1; V.CZ = V.Z + 1;
  V.X1 = V.X - 1; V.Y1 = V.Y - 1; V.Z1 = V.Z - 1;
  for (int k = 0; k < 3; ++k) {
    V.lo[k] = (long long)llrint((-0.5 - 1e-6) * kFix);
    V.hi[k] = (long long)llrint(((double)vol->dims[k] - 0.5 + 1e-6) * kFix);
    V.top[k] = (long long)(vol->dims[k] - 1) << 32;
    V.bmin[k] = vol->box_min[k];
    V.bmax[k] = vol->box_max[k];
    V.scale[k] = (double)vol->dims[k] / (vol->box_max[k] - vol->box_min[k]);
  }
  G.cams = cams; G.dt = p->dt; G.dt32 = (float)p->dt;
  G.W = p->width; G.H = p->height; G.row0 = 0; G.row1 = p->height;
  const dim3 grid((G.W + SW - 1) / SW, (G.H + SH - 1) / SH, n_views);
  const size_t sm = CAP * 2 * sizeof(float4);
  cudaStream_t st = (cudaStream_t)stream;
#define RUNK(KK)                                                                        \
  if (K == KK) {                                                                        \
    cudaFuncSetAttribute(probe_staged_kernel<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)sm);                                                      \
    probe_staged_kernel<KK><<<grid, SNT, sm, st>>>(V, G, lin, out, stats);               \
  }
  RUNK(8) RUNK(16) RUNK(32)
#undef RUNK
  return (int)cudaGetLastError();
}

extern "C" int sm_run(const ddvr_volume* vol, const ddvr_camera* cams, int n_views,
                      const ddvr_params* p, const float* lin, unsigned* ctr, float* out,
                      int ctas_per_sm, void* stream) {
  VolArgs V;
  Geometry G;
  V.X = vol->dims[0]; V.Y = vol->dims[1]; V.Z = vol->dims[2];
  V.YZ = V.Y * V.Z; V.CY = V.Y + 1; V.CZ = V.Z + 1;
  V.X1 = V.X - 1; V.Y1 = V.Y - 1; V.Z1 = V.Z - 1;
  for (int k = 0; k < 3; ++k) {
    V.lo[k] = (long long)llrint((-0.5 - 1e-6) * kFix);
    V.hi[k] = (long long)llrint(((double)vol->dims[k] - 0.5 + 1e-6) * kFix);
    V.top[k] = (long long)(vol->dims[k] - 1) << 32;
    V.bmin[k] = vol->box_min[k];
    V.bmax[k] = vol->box_max[k];
    V.scale[k] = (double)vol->dims[k] / (vol->box_max[k] - vol->box_min[k]);
  }
  G.cams = cams; G.dt = p->dt; G.dt32 = (float)p->dt;
  G.W = p->width; G.H = p->height; G.row0 = 0; G.row1 = p->height;
  const int tx = (G.W + kTile - 1) / kTile, ty = (G.H + kTile - 1) / kTile;
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemsetAsync(ctr, 0, 148 * sizeof(unsigned), st);
  probe_sm_kernel<<<148 * ctas_per_sm, kThreads, 0, st>>>(V, G, lin, tx, ty, tx * ty * n_views,
                                                           148, ctr, out);
  return (int)cudaGetLastError();
}

extern "C" int brick_run(const ddvr_volume* vol, const ddvr_camera* cams, int n_views,
                         const ddvr_params* p, int brick, const float* lin, float* bricks,
                         float* out, int rebrick, void* stream) {
  VolArgs V;
  Geometry G;
  // minimal copies of make_vol / make_geo for the probe (fields the march reads)
  V.X = vol->dims[0]; V.Y = vol->dims[1]; V.Z = vol->dims[2];
  V.YZ = V.Y * V.Z; V.CY = V.Y + 1; V.CZ = V.Z + 1;
  V.X1 = V.X - 1; V.Y1 = V.Y - 1; V.Z1 = V.Z - 1;
  for (int k = 0; k < 3; ++k) {
    V.lo[k] = (long long)llrint((-0.5 - 1e-6) * kFix);
    V.hi[k] = (long long)llrint(((double)vol->dims[k] - 0.5 + 1e-6) * kFix);
    V.top[k] = (long long)(vol->dims[k] - 1) << 32;
    V.bmin[k] = vol->box_min[k];
    V.bmax[k] = vol->box_max[k];
    V.scale[k] = (double)vol->dims[k] / (vol->box_max[k] - vol->box_min[k]);
  }
  G.cams = cams;
  G.dt = p->dt;
  G.dt32 = (float)p->dt;
  G.W = p->width; G.H = p->height; G.row0 = 0; G.row1 = p->height;
  const int CX = V.X + 1, NBY = (V.CY + 1) / 2, NBZ = (V.CZ + 1) / 2;
  cudaStream_t st = (cudaStream_t)stream;
  if (rebrick) {
    const long long n = (long long)CX * V.CY * V.CZ;
    rebrick_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(lin, CX, V.CY, V.CZ, NBY, NBZ,
                                                                bricks);
  }
  const dim3 grid((G.W + kTile - 1) / kTile, (G.H + kTile - 1) / kTile, n_views);
  if (brick) probe_kernel<true><<<grid, kThreads, 0, st>>>(V, G, bricks, NBY, NBZ, out);
  else probe_kernel<false><<<grid, kThreads, 0, st>>>(V, G, lin, NBY, NBZ, out);
  return (int)cudaGetLastError();
}
