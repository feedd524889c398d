// Internal-node assembly for the block formulation of the node step
// (solver.py:138-165):
//
//   Z = I + W G = [[I, X], [Y, I]],  X = B H_r,  Y = B^T H_l   (solver.py:142-148)
//
// is eliminated with its identity (1,1) block as pivot; the only pivoted LU is
// that of S = I - Y X (linalg.py:199-213 on the Schur complement, pivots among
// its rows). The augmented matrix handed to the LU kernels is
//
//   Aug = [[S, E], [F, C]],  E = P_r^T - Y P_l^T,  F = P_l H_l X - P_r H_r,  C = P_l H_l P_l^T
//
// and after the LU its trailing block is C - F S^-1 E = P G Z^-1 P^T = H
// (solver.py:154-164). X, Y, P_l H_l and the products are DMMA GEMMs
// (factorize.cu); this file holds the element-wise pieces: the Gaussian
// coupling block, the S = I and E = P_r^T initial blocks, the padded P copy,
// ||Z||_1, the composed row interchanges and H = sym(trailing block).
#include <algorithm>

#include "gauss.cuh"
#include "gemm.cuh"
#include "kernels.cuh"

namespace ks {

// Coupling B = K(S_l, S_r) (compress.py:281-283) and its transpose, zero
// padded to s_pad^2: grid.z = 2 x nodes, the second half evaluates
// K(S_r, S_l) into B^T (the difference form is symmetric bit for bit).
__global__ void __launch_bounds__(256) k_coupling(DevTree t, NodeBatch nb) {
  pdl_wait();
  const bool tr = blockIdx.z >= (unsigned)nb.count;
  const int k = tr ? blockIdx.z - nb.count : blockIdx.z;
  const int l = tr ? nb.right[k] : nb.left[k], r = tr ? nb.left[k] : nb.right[k];
  const int sl = t.rank[l], sr = t.rank[r];
  const int r0 = blockIdx.y * GT, c0 = blockIdx.x * GT;
  double sq[4][4];
  gauss_tile<true>(t, t.skel_pos + t.skel_off[l], 0, sl, t.skel_pos + t.skel_off[r], 0, sr, r0, c0, sq);
  const double den = -2.0 * t.h * t.h;
  double* B = (tr ? nb.BcT : nb.Bc) + (int64_t)k * nb.s_pad * nb.s_pad;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = r0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c0 + tx + 16 * j;
      B[(int64_t)rr * nb.s_pad + cc] = (rr < sl && cc < sr) ? exp(sq[i][j] / den) : 0.0;
    }
  }
}

// GEMM form for large d: the skeleton coordinates of both children gathered
// into XS (zt rows of dk per node: [left; right], zero padded) with their
// squared norms, then B = K(S_l, S_r) and B^T = K(S_r, S_l) as one grouped
// DMMA Gram GEMM with the Gaussian epilogue (gemm.cuh EPI 4). The two products
// sum the same terms in the same order, so B^T is B transposed bit for bit.
__global__ void __launch_bounds__(256) k_gather_skel(DevTree t, NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.y, row = blockIdx.x;  // row < zt
  const int S = nb.s_pad, dk = nb.dk;
  const bool right = row >= S;
  const int v = right ? nb.right[k] : nb.left[k], i = right ? row - S : row;
  const int rk = t.rank[v];
  double* out = nb.XS + ((int64_t)k * nb.zt + row) * dk;
  __shared__ double red[8];
  double s = 0.0;
  if (i < rk) {
    const double* x = t.coords + (int64_t)t.skel_pos[t.skel_off[v] + i] * t.d;
    for (int c = threadIdx.x; c < dk; c += 256) {
      const double xv = c < t.d ? x[c] : 0.0;
      out[c] = xv;
      s = fma(xv, xv, s);
    }
  } else {
    for (int c = threadIdx.x; c < dk; c += 256) out[c] = 0.0;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    nb.XN[(int64_t)k * nb.zt + row] = tot;
  }
}

void launch_coupling(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  if (nb.XS) {
    launch_pdl(k_gather_skel, dim3(nb.zt, nb.count), dim3(256), 0, st, t, nb);
    const int S = nb.s_pad, dk = nb.dk;
    const int64_t XSS = (int64_t)nb.zt * dk, SS = (int64_t)S * S;
    GemmGroup gg{};
    gg.count = 2;
    for (int p = 0; p < 2; ++p) {
      GemmArgs& g = gg.p[p];
      g.M = S; g.N = S; g.K = dk; g.batch = nb.count;
      g.A = Operand{nb.XS + (p ? (int64_t)S * dk : 0), dk, XSS, nullptr};
      g.B = Operand{nb.XS + (p ? 0 : (int64_t)S * dk), dk, XSS, nullptr};
      g.C = OperandW{p ? nb.BcT : nb.Bc, S, SS, nullptr};
      g.alpha = 1.0; g.beta = 0.0; g.tri = 0;
      g.ce = CoupEpi{nb.XN + (p ? S : 0), nb.XN + (p ? 0 : S), nb.zt, p ? nb.right : nb.left,
                     p ? nb.left : nb.right, t.rank, 1.0 / (-2.0 * t.h * t.h)};
    }
    gemm_group_coupling(gg, st);
    return;
  }
  dim3 g(nb.s_pad / GT, nb.s_pad / GT, 2 * nb.count);
  launch_pdl(k_coupling, g, dim3(256), 0, st, t, nb);
}

// Padded candidate index i' of a node's P row maps to the reference's cand
// index (cand = [skel_l; skel_r], compress.py:213): i' < s_pad -> i' (if < s_l),
// i' >= s_pad -> s_l + (i' - s_pad) (if < s_r).
__device__ __forceinline__ int cand_index(int i, int S, int sl, int sr) {
  return (i < S) ? (i < sl ? i : -1) : (i - S < sr ? sl + (i - S) : -1);
}

// The operator's P of every internal node in the two layouts the assembly
// GEMMs and the solve read (they depend only on the operator, not on lambda:
// written by the first factorization of a handle, kept afterwards):
// Pn, one CTA per row j: P[j][cand(i)] for the padded candidate index i
__global__ void __launch_bounds__(256) k_pn_layout(DevTree t, NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.y, j = blockIdx.x;
  const int S = nb.s_pad, ZT = nb.zt;
  const int v = nb.node[k], sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]], sv = t.rank[v];
  const double* P = t.coeff + t.coeff_off[v] + (int64_t)j * (sl + sr);
  double* out = nb.Pn + (int64_t)k * S * ZT + (int64_t)j * ZT;
  for (int i = threadIdx.x; i < ZT; i += 256) {
    const int ci = cand_index(i, S, sl, sr);
    out[i] = (ci >= 0 && j < sv) ? P[ci] : 0.0;
  }
}

// P^T (zt x S: rows [0, S) P_l^T, rows [S, 2S) P_r^T) through 32 x 32
// shared-memory tiles: reads along P's rows, writes along P^T's
__global__ void __launch_bounds__(256) k_pt_layout(DevTree t, NodeBatch nb) {
  pdl_wait();
  __shared__ double tile[32][33];
  const int k = blockIdx.z;
  const int S = nb.s_pad;
  const int v = nb.node[k], sl = t.rank[nb.left[k]], sr = t.rank[nb.right[k]], sv = t.rank[v];
  const double* P = t.coeff + t.coeff_off[v];
  const int cand = sl + sr;
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;  // j: P row (parent skeleton), i: padded cand index
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  {
    const int ci = cand_index(i0 + tx, S, sl, sr);
    for (int jj = ty; jj < 32; jj += 8) {
      const int j = j0 + jj;
      tile[jj][tx] = (ci >= 0 && j < sv) ? P[(int64_t)j * cand + ci] : 0.0;
    }
  }
  __syncthreads();
  double* PT = nb.PT + (int64_t)k * nb.zt * S;
  for (int ii = ty; ii < 32; ii += 8) PT[(int64_t)(i0 + ii) * S + j0 + tx] = tile[tx][ii];
}

void launch_p_layout(const DevTree& t, const NodeBatch& nb, cudaStream_t st) {
  launch_pdl(k_pn_layout, dim3(nb.s_pad, nb.count), dim3(256), 0, st, t, nb);
  launch_pdl(k_pt_layout, dim3(nb.s_pad / 32, nb.zt / 32, nb.count), dim3(256), 0, st, t, nb);
}

// ||Z||_1 = max column abs sum of [[I, X], [Y, I]] (linalg.py:176): the columns
// of the left child's block are 1 + |Y| column sums, the right child's 1 + |X|
// column sums (padded columns give 1, never above a real column's sum). 32
// columns per CTA, rows split over 8 warps; the max goes through an integer
// atomicMax on the non-negative double's bit pattern (norm1 zeroed first).
__global__ void __launch_bounds__(256) k_znorm1(NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.y, S = nb.s_pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;  // Z column, < 2S
  const double* M = nb.XY + (int64_t)k * 2 * S * S + (c < S ? (int64_t)S * S : 0);  // Y for c < S, else X
  const int col = c < S ? c : c - S;
  __shared__ double red[8][33];
  double s = 0.0;
#pragma unroll 8
  for (int i = warp; i < S; i += 8) s += fabs(M[(int64_t)i * S + col]);
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double tot = 1.0;
    for (int w = 0; w < 8; ++w) tot += red[w][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot = fmax(tot, __shfl_xor_sync(0xffffffffu, tot, o));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(nb.norm1 + k), __double_as_longlong(tot));
  }
}

void launch_znorm1(const NodeBatch& nb, cudaStream_t st) {
  cudaMemsetAsync(nb.norm1, 0, sizeof(double) * nb.count, st);
  launch_pdl(k_znorm1, dim3(2 * nb.s_pad / 32, nb.count), dim3(256), 0, st, nb);
}

// Composed row interchanges of the S LU (pm: (Pi v)[i] = v[pm[i]]) for the solve.
__global__ void __launch_bounds__(1024) k_compose_perm(NodeBatch nb) {
  pdl_wait();
  const int k = blockIdx.x;
  const int TP = nb.t_pad;
  const int* piv = nb.piv + (int64_t)k * TP;
  int* pm = nb.pm + (int64_t)k * TP;
  extern __shared__ __align__(16) int ps[];
  for (int i = threadIdx.x; i < TP; i += blockDim.x) ps[i] = piv[i];
  __syncthreads();
  // every thread follows one row through the swap sequence: the row that
  // starts at r ends at f(r), so pm[f(r)] = r (same result as swapping pm);
  // t_pad is a multiple of 64, the swaps are read four at a time
  for (int r = threadIdx.x; r < TP; r += blockDim.x) {
    int f = r;
    const int4* p4 = reinterpret_cast<const int4*>(ps);
    for (int i = 0; i < TP / 4; ++i) {
      const int4 q = p4[i];
      const int i0 = 4 * i;
      f = (f == i0) ? q.x : (f == q.x ? i0 : f);
      f = (f == i0 + 1) ? q.y : (f == q.y ? i0 + 1 : f);
      f = (f == i0 + 2) ? q.z : (f == q.z ? i0 + 2 : f);
      f = (f == i0 + 3) ? q.w : (f == q.w ? i0 + 3 : f);
    }
    pm[f] = r;
  }
}

void launch_compose_perm(const NodeBatch& nb, cudaStream_t st) {
  launch_pdl(k_compose_perm, dim3(nb.count), dim3(std::min(1024, nb.t_pad)), sizeof(int) * nb.t_pad, st, nb);
}

// H = sym(trailing block) -> Hbuf[node] (solver.py:163): 32 x 32 tiles, the
// transposed tile through shared memory so both reads run along rows.
__global__ void __launch_bounds__(256) k_extract_h(NodeBatch nb, double* H, int64_t stride) {
  pdl_wait();
  __shared__ double tt[32][33];
  const int k = blockIdx.z;
  const int S = nb.s_pad, T = nb.T, TP = nb.t_pad;
  const double* A = nb.Aug + (int64_t)k * T * T + (int64_t)TP * T + TP;
  double* h = H + (int64_t)nb.node[k] * stride;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) tt[r][tx] = A[(int64_t)(j0 + r) * T + i0 + tx];  // A[j][i]
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    h[(int64_t)i * S + j] = 0.5 * (A[(int64_t)i * T + j] + tt[tx][r]);
  }
}

void launch_extract_h(const NodeBatch& nb, double* H, int64_t h_stride, cudaStream_t st) {
  launch_pdl(k_extract_h, dim3(nb.s_pad / 32, nb.s_pad / 32, nb.count), dim3(256), 0, st, nb, H, h_stride);
}

}  // namespace ks
