// k_mesh.cu — NEXT-3: O on a lattice, Marching Cubes, per-vertex normals.
//
// PAPER.md:L680 (§4.1): "we first evaluate O(q) at 512-resolution grid points. Then, we use Marching
// Cubes on the resulting grid"; PAPER.md:L962-971 (§4.5): "we reconstruct the mesh in our
// representation and obtain the normals using a single forward pass" (Eq. func-normal).
//
// Lattice: N^3 nodes, node n = i + N (j + N k) at lo + (hi - lo) * (i, j, k) / (N - 1) (x fastest).
// A node is "inside" iff O < iso. Vertices sit on the lattice edges whose end nodes differ
// (linear interpolation of O); each node owns the vertices of its +x, +y, +z edges, so a vertex is
// emitted once and shared by the (up to 4) cubes around its edge: an indexed, watertight mesh.
//
// The triangle table (256 cases) is generated on the host from the cube's faces rather than typed in:
// on every face the iso-curve is a set of segments joining the face's sign-changing edges; on a face
// with four such edges (diagonal inside corners) the segments separate the inside corners. The rule
// depends only on the face's four corners, so the two cubes sharing a face draw the same segments
// and the surface is closed. Segments are oriented (inside on the left, seen from outside the
// cube), chained into loops through the edge points, and every loop is fanned into triangles whose
// right-hand normal points from inside (O < iso) to outside.
#include <algorithm>
#include <cstring>
#include <vector>

#include "k_common.cuh"

namespace ef {

__constant__ int8_t c_mc_tri[256][16];  // edge ids, 3 per triangle, -1 terminated
__constant__ uint8_t c_mc_ntri[256];

// cube corner v = x + 2y + 4z; edge e = 4 a + idx along axis a, idx = the other two coordinates
// (a = 0: y + 2z; a = 1: x + 2z; a = 2: x + 2y), from its low corner to its high corner
static void edge_corners(int e, int& c0, int& c1) {
  const int a = e >> 2, idx = e & 3;
  int x = 0, y = 0, z = 0;
  if (a == 0) { y = idx & 1; z = idx >> 1; }
  if (a == 1) { x = idx & 1; z = idx >> 1; }
  if (a == 2) { x = idx & 1; y = idx >> 1; }
  c0 = x + 2 * y + 4 * z;
  c1 = c0 + (1 << a);
}

static int edge_of(int c0, int c1) {
  if (c0 > c1) std::swap(c0, c1);
  const int d = c1 - c0, a = d == 1 ? 0 : (d == 2 ? 1 : 2);
  const int x = c0 & 1, y = (c0 >> 1) & 1, z = (c0 >> 2) & 1;
  const int idx = a == 0 ? y + 2 * z : (a == 1 ? x + 2 * z : x + 2 * y);
  return 4 * a + idx;
}

struct McTable {
  int8_t tri[256][16];
  uint8_t ntri[256];
};

static void mc_build_table(McTable& T) {
  std::memset(T.tri, -1, sizeof(T.tri));
  std::memset(T.ntri, 0, sizeof(T.ntri));
  // the 6 faces, corners counter-clockwise seen from outside: axis a, side s, (u, w, a) right-handed
  int face[6][4];
  for (int a = 0; a < 3; ++a) {
    const int u = (a + 1) % 3, w = (a + 2) % 3;
    for (int s = 0; s < 2; ++s) {
      const int uw[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
      for (int k = 0; k < 4; ++k) {
        const int kk = s ? k : (4 - k) % 4;  // the -a face runs the other way round
        int c = s << a;
        c |= uw[kk][0] << u;
        c |= uw[kk][1] << w;
        face[2 * a + s][k] = c;
      }
    }
  }
  auto corner_pos = [](int c, float* p) {
    p[0] = (float)(c & 1); p[1] = (float)((c >> 1) & 1); p[2] = (float)((c >> 2) & 1);
  };
  for (int cs = 0; cs < 256; ++cs) {
    auto in = [&](int c) { return (cs >> c) & 1; };
    int next[12];
    for (int e = 0; e < 12; ++e) next[e] = -1;
    for (int f = 0; f < 6; ++f) {
      int order[4], type[4], m = 0;
      for (int k = 0; k < 4; ++k) {
        const int c0 = face[f][k], c1 = face[f][(k + 1) % 4];
        if (in(c0) != in(c1)) {
          order[m] = edge_of(c0, c1);
          type[m] = in(c0) ? 1 : 0;  // 1: exit (inside -> outside along the CCW walk), 0: enter
          ++m;
        }
      }
      // pair every exit with the cyclically preceding enter (separates inside corners)
      for (int k = 0; k < m; ++k) {
        if (type[k] != 1) continue;
        const int p = (k + m - 1) % m;
        next[order[k]] = order[p];
      }
    }
    // chain the loops and fan them into triangles
    bool used[12] = {false};
    int nt = 0;
    for (int e0 = 0; e0 < 12; ++e0) {
      if (next[e0] < 0 || used[e0]) continue;
      std::vector<int> loop;
      for (int e = e0; !used[e]; e = next[e]) {
        used[e] = true;
        loop.push_back(e);
      }
      for (size_t k = 1; k + 1 < loop.size(); ++k) {
        T.tri[cs][3 * nt] = (int8_t)loop[0];
        T.tri[cs][3 * nt + 1] = (int8_t)loop[k];
        T.tri[cs][3 * nt + 2] = (int8_t)loop[k + 1];
        ++nt;
      }
    }
    T.ntri[cs] = (uint8_t)nt;
  }
  // orientation: case 1 (corner 0 inside) must have its normal pointing away from corner 0
  float p[3][3];
  for (int k = 0; k < 3; ++k) {
    int c0, c1;
    edge_corners(T.tri[1][k], c0, c1);
    float a[3], b[3];
    corner_pos(c0, a);
    corner_pos(c1, b);
    for (int d = 0; d < 3; ++d) p[k][d] = 0.5f * (a[d] + b[d]);
  }
  const float u[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
  const float v[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
  const float nrm = (u[1] * v[2] - u[2] * v[1]) + (u[2] * v[0] - u[0] * v[2]) + (u[0] * v[1] - u[1] * v[0]);
  if (nrm < 0.0f) {
    for (int cs = 0; cs < 256; ++cs)
      for (int t = 0; t < T.ntri[cs]; ++t) std::swap(T.tri[cs][3 * t + 1], T.tri[cs][3 * t + 2]);
  }
}

static bool g_mc_ready = false;

int mc_max_tris_per_cube() {
  McTable T;
  mc_build_table(T);
  int mx = 0;
  for (int cs = 0; cs < 256; ++cs) mx = std::max(mx, (int)T.ntri[cs]);
  return mx;
}

cudaError_t mc_upload_table() {
  if (g_mc_ready) return cudaSuccess;  // (per process; the library serves one device per handle)
  McTable T;
  mc_build_table(T);
  cudaError_t e = cudaMemcpyToSymbol(c_mc_tri, T.tri, sizeof(T.tri));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_mc_ntri, T.ntri, sizeof(T.ntri));
  if (e == cudaSuccess) g_mc_ready = true;
  return e;
}

void mc_table_host(int8_t* tri /*256*16*/, uint8_t* ntri /*256*/) {
  McTable T;
  mc_build_table(T);
  std::memcpy(tri, T.tri, sizeof(T.tri));
  std::memcpy(ntri, T.ntri, sizeof(T.ntri));
}

// ---------------------------------------------------------------------------------- device
__global__ void k_lattice_q(int N, float lx, float ly, float lz, float sx, float sy, float sz, int k0, int nk,
                            float* __restrict__ q) {
  const int64_t per = (int64_t)N * N;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < per * nk; p += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(p % N), j = (int)((p / N) % N), k = k0 + (int)(p / per);
    q[3 * p] = fmaf((float)i, sx, lx);
    q[3 * p + 1] = fmaf((float)j, sy, ly);
    q[3 * p + 2] = fmaf((float)k, sz, lz);
  }
}

int launch_lattice_q(int N, const float* lo, const float* step, int k0, int nk, float* q, cudaStream_t s) {
  const int64_t n = (int64_t)N * N * nk;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_lattice_q<<<(unsigned)blocks, 256, 0, s>>>(N, lo[0], lo[1], lo[2], step[0], step[1], step[2], k0, nk, q);
  return 1;
}

// per node: the sign-changing edges it owns (+x, +y, +z bits) and their count
__global__ void k_mc_nodes(const float* __restrict__ O, int N, float iso, uint8_t* __restrict__ mask,
                           uint32_t* __restrict__ cnt) {
  const int64_t n3 = (int64_t)N * N * N, NN = (int64_t)N * N;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n3; n += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(n % N), j = (int)((n / N) % N), k = (int)(n / NN);
    const bool s = O[n] < iso;
    uint32_t m = 0;
    if (i + 1 < N && ((O[n + 1] < iso) != s)) m |= 1u;
    if (j + 1 < N && ((O[n + N] < iso) != s)) m |= 2u;
    if (k + 1 < N && ((O[n + NN] < iso) != s)) m |= 4u;
    mask[n] = (uint8_t)m;
    cnt[n] = __popc(m);
  }
}

__device__ __forceinline__ uint32_t mc_case(const float* __restrict__ O, int64_t n, int64_t N, int64_t NN, float iso) {
  uint32_t cs = 0;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int64_t m = n + (v & 1) + ((v >> 1) & 1) * N + ((v >> 2) & 1) * NN;
    cs |= (O[m] < iso ? 1u : 0u) << v;
  }
  return cs;
}

// per cube (indexed by its low node, cubes of the last layer count 0): triangles of its case
__global__ void k_mc_cubes(const float* __restrict__ O, int N, float iso, uint32_t* __restrict__ cnt) {
  const int64_t n3 = (int64_t)N * N * N, NN = (int64_t)N * N;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n3; n += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(n % N), j = (int)((n / N) % N), k = (int)(n / NN);
    uint32_t t = 0;
    if (i + 1 < N && j + 1 < N && k + 1 < N) t = c_mc_ntri[mc_case(O, n, N, NN, iso)];
    cnt[n] = t;
  }
}

__global__ void k_mc_verts(const float* __restrict__ O, int N, float iso, float lx, float ly, float lz, float sx,
                           float sy, float sz, const uint8_t* __restrict__ mask, const uint32_t* __restrict__ voff,
                           float* __restrict__ verts) {
  const int64_t n3 = (int64_t)N * N * N, NN = (int64_t)N * N;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n3; n += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t m = mask[n];
    if (!m) continue;
    const int i = (int)(n % N), j = (int)((n / N) % N), k = (int)(n / NN);
    const float px = fmaf((float)i, sx, lx), py = fmaf((float)j, sy, ly), pz = fmaf((float)k, sz, lz);
    const float v0 = O[n];
    uint32_t out = voff[n];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (!((m >> a) & 1u)) continue;
      const float v1 = O[n + (a == 0 ? 1 : (a == 1 ? N : NN))];
      const float t = (iso - v0) / (v1 - v0);  // linear interpolation along the edge
      float* p = verts + 3 * (size_t)out;
      p[0] = a == 0 ? fmaf(t, sx, px) : px;
      p[1] = a == 1 ? fmaf(t, sy, py) : py;
      p[2] = a == 2 ? fmaf(t, sz, pz) : pz;
      ++out;
    }
  }
}

__global__ void k_mc_tris(const float* __restrict__ O, int N, float iso, const uint8_t* __restrict__ mask,
                          const uint32_t* __restrict__ voff, const uint32_t* __restrict__ toff,
                          int32_t* __restrict__ tris) {
  const int64_t n3 = (int64_t)N * N * N, NN = (int64_t)N * N;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n3; n += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(n % N), j = (int)((n / N) % N), k = (int)(n / NN);
    if (i + 1 >= N || j + 1 >= N || k + 1 >= N) continue;
    const uint32_t cs = mc_case(O, n, N, NN, iso);
    const int nt = c_mc_ntri[cs];
    uint32_t out = toff[n];
    for (int t = 0; t < 3 * nt; ++t) {
      const int e = c_mc_tri[cs][t], a = e >> 2, idx = e & 3;
      // the edge's low node: the cube's low node + the edge's offsets in the other two axes
      int64_t node = n;
      if (a == 0) node += (idx & 1) * (int64_t)N + (idx >> 1) * NN;
      if (a == 1) node += (idx & 1) + (idx >> 1) * NN;
      if (a == 2) node += (idx & 1) + (idx >> 1) * (int64_t)N;
      const uint32_t m = mask[node];
      tris[3 * (size_t)out + t] = (int32_t)(voff[node] + __popc(m & ((1u << a) - 1u)));
    }
  }
}

__global__ void k_normalize3(float* __restrict__ v, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const float x = v[3 * p], y = v[3 * p + 1], z = v[3 * p + 2];
    const float r = sqrtf(fmaf(x, x, fmaf(y, y, z * z)));
    const float inv = r > 0.0f ? 1.0f / r : 0.0f;
    v[3 * p] = x * inv;
    v[3 * p + 1] = y * inv;
    v[3 * p + 2] = z * inv;
  }
}

static unsigned grid_n(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

int launch_mc_count(const float* O, int N, float iso, uint8_t* mask, uint32_t* vcnt, uint32_t* tcnt, cudaStream_t s) {
  const int64_t n3 = (int64_t)N * N * N;
  k_mc_nodes<<<grid_n(n3), 256, 0, s>>>(O, N, iso, mask, vcnt);
  k_mc_cubes<<<grid_n(n3), 256, 0, s>>>(O, N, iso, tcnt);
  return 2;
}

int launch_mc_emit(const float* O, int N, float iso, const float* lo, const float* step, const uint8_t* mask,
                   const uint32_t* voff, const uint32_t* toff, float* verts, int32_t* tris, cudaStream_t s) {
  const int64_t n3 = (int64_t)N * N * N;
  k_mc_verts<<<grid_n(n3), 256, 0, s>>>(O, N, iso, lo[0], lo[1], lo[2], step[0], step[1], step[2], mask, voff, verts);
  k_mc_tris<<<grid_n(n3), 256, 0, s>>>(O, N, iso, mask, voff, toff, tris);
  return 2;
}

int launch_normalize3(float* v, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  k_normalize3<<<grid_n(n), 256, 0, s>>>(v, n);
  return 1;
}

}  // namespace ef
