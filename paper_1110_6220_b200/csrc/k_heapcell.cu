// Kernel (3): the heap-cell methods HCM / FHCM (/root/reference/proj/src/
// heap_cell.cpp:13-336) as a device-resident exact replay.
//
// One warp runs the reference's loop: lane 0 owns an indexed binary min-heap
// of cells keyed by (cell value, cell id) (indexed_min_heap.hpp, ties to the
// smaller id), the whole warp processes the popped cell in shared memory --
// border snapshot, reset_locks, locking sweeps in anti-diagonal wavefront
// order (bit-identical to the row-by-row loop including every counter,
// SURVEY.md finding 7), the four border scans with warp reductions -- and
// lane 0 applies the scans to the heap.  The pop sequence, and therefore
// every value and counter, is the reference's.  FHCM's output depends on that
// exact order (SURVEY.md finding 6), which is why the replay is exact rather
// than band-parallel.
#include "eik_internal.h"
#include "k_common.cuh"

namespace eikb200 {

namespace {

enum { SW = 0, NW = 1, NE = 2, SE = 3 };
enum { WEST = 0, EAST = 1, SOUTH = 2, NORTH = 3 };
__device__ const int kFlagOrder[4] = {NE, NW, SE, SW};  // heap_cell.cpp:13-14
__device__ const int kRotation[4] = {SW, NW, NE, SE};   // heap_cell.cpp:15-16

// ---- indexed min-heap (single thread) -------------------------------------
struct DevHeap {
  double* key;
  int* pos;
  int* arr;
  int size;
  __device__ bool less(int a, int b) const {
    const double ka = key[a], kb = key[b];
    if (ka != kb) return ka < kb;
    return a < b;
  }
  __device__ void up(int p) {
    const int id = arr[p];
    while (p > 0) {
      const int par = (p - 1) >> 1;
      if (!less(id, arr[par])) break;
      arr[p] = arr[par];
      pos[arr[p]] = p;
      p = par;
    }
    arr[p] = id;
    pos[id] = p;
  }
  __device__ void down(int p) {
    const int id = arr[p];
    for (;;) {
      int c = 2 * p + 1;
      if (c >= size) break;
      if (c + 1 < size && less(arr[c + 1], arr[c])) ++c;
      if (!less(arr[c], id)) break;
      arr[p] = arr[c];
      pos[arr[p]] = p;
      p = c;
    }
    arr[p] = id;
    pos[id] = p;
  }
  __device__ bool contains(int id) const { return pos[id] >= 0; }
  __device__ void insert(int id, double k) {
    key[id] = k;
    pos[id] = size;
    arr[size++] = id;
    up(pos[id]);
  }
  __device__ void decrease(int id, double k) {
    key[id] = k;
    up(pos[id]);
  }
  __device__ int pop() {
    const int top = arr[0];
    const int last = arr[--size];
    pos[top] = -1;
    if (size > 0) {
      arr[0] = last;
      pos[last] = 0;
      down(0);
    }
    return top;
  }
};

struct HTile {
  double* U;      // (h+2) x pu values with cross halo
  double* Ct;     // (h+2) x pu costs with halo (-1 = exit / off-grid)
  uint8_t* lock;  // h x w, 1 = unlocked
  int pu, w, h;
  __device__ double& u(int x, int y) const { return U[(y + 1) * pu + (x + 1)]; }
  __device__ double c(int x, int y) const { return Ct[(y + 1) * pu + (x + 1)]; }
};

// reset_locks (heap_cell.cpp:65-94)
__device__ void reset_locks(const HTile& T, bool west_in, bool east_in, bool south_in,
                            bool north_in, int lane) {
  for (int k = lane; k < T.w * T.h; k += 32) {
    const int y = k / T.w, x = k % T.w;
    bool un = false;
    if (T.c(x, y) >= 0.0) {
      un = (west_in && x == 0) || (east_in && x == T.w - 1) || (south_in && y == 0) ||
           (north_in && y == T.h - 1);
      un = un || (x + 1 < T.w && T.c(x + 1, y) < 0.0) || (x > 0 && T.c(x - 1, y) < 0.0) ||
           (y + 1 < T.h && T.c(x, y + 1) < 0.0) || (y > 0 && T.c(x, y - 1) < 0.0);
    }
    T.lock[k] = un ? 1 : 0;
  }
  __syncwarp();
}

// locked_sweep (heap_cell.cpp:98-126) in anti-diagonal order
__device__ bool locked_sweep(const HTile& T, int dir, int lane, long long& updates) {
  const bool iasc = (dir == SW || dir == NW);
  const bool jasc = (dir == SW || dir == SE);
  bool changed = false;
  const int nsteps = T.w + T.h - 1;
  for (int s = 0; s < nsteps; ++s) {
    for (int b = lane; b < T.h; b += 32) {
      const int a = s - b;
      if (a >= 0 && a < T.w) {
        const int x = iasc ? a : T.w - 1 - a;
        const int y = jasc ? b : T.h - 1 - b;
        uint8_t* lk = T.lock + y * T.w + x;
        if (*lk) {
          *lk = 0;
          ++updates;
          double* p = &T.u(x, y);
          const double cand = node_update4(p[1], p[-1], p[T.pu], p[-T.pu], T.c(x, y));
          if (cand < *p) {
            *p = cand;
            changed = true;
            // unlock in-cell neighbours that this value can still improve
            if (x + 1 < T.w && T.c(x + 1, y) >= 0.0 && p[1] > cand) lk[1] = 1;
            if (x > 0 && T.c(x - 1, y) >= 0.0 && p[-1] > cand) lk[-1] = 1;
            if (y + 1 < T.h && T.c(x, y + 1) >= 0.0 && p[T.pu] > cand) lk[T.w] = 1;
            if (y > 0 && T.c(x, y - 1) >= 0.0 && p[-T.pu] > cand) lk[-T.w] = 1;
          }
        }
      }
    }
    __syncwarp();
  }
  return __any_sync(kFull, changed);
}

struct Scan {
  bool add;
  unsigned fl;
  double cand;
  bool mon_checked, mon_single;
};

__device__ void mono_sides(int from_side, int out[2]) {  // cells.cpp:49-60
  switch (from_side) {
    case WEST: out[0] = NW; out[1] = SW; break;
    case EAST: out[0] = NE; out[1] = SE; break;
    case SOUTH: out[0] = SW; out[1] = SE; break;
    default: out[0] = NW; out[1] = NE; break;
  }
}

// scan_cell_boundary (heap_cell.cpp:173-239) as warp reductions
__device__ Scan scan_side(const HcArgs& a, const HTile& T, int side, const double* before,
                          bool first_removal, int64_t ib, int64_t jb, int cx, int cy, int lane) {
  const bool vertical = (side == WEST || side == EAST);
  const int len = vertical ? T.h : T.w;
  double vmax = -kInf;
  int arg = 0x7fffffff;
  bool add = false, inc_viol = false, dec_viol = false;
  for (int t = lane; t < len; t += 32) {
    int x, y, ax, ay;
    switch (side) {
      case WEST: x = 0; y = t; ax = -1; ay = t; break;
      case EAST: x = T.w - 1; y = t; ax = T.w; ay = t; break;
      case SOUTH: x = t; y = 0; ax = t; ay = -1; break;
      default: x = t; y = T.h - 1; ax = t; ay = T.h; break;
    }
    const double vi = T.u(x, y);
    if (vi > vmax) {  // first strict maximum along the strip
      vmax = vi;
      arg = t;
    }
    const bool across_exit = T.c(ax, ay) < 0.0;
    const bool changed = vi < before[t];
    if (!across_exit && vi < T.u(ax, ay) && (changed || (first_removal && T.c(x, y) < 0.0)))
      add = true;
    if (t > 0) {
      const double prev = vertical ? T.u(x, y - 1) : T.u(x - 1, y);
      if (vi < prev) inc_viol = true;
      if (vi > prev) dec_viol = true;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(kFull, vmax, o);
    const int oa = __shfl_xor_sync(kFull, arg, o);
    if (ov > vmax || (ov == vmax && oa < arg)) {
      vmax = ov;
      arg = oa;
    }
  }
  Scan r;
  r.add = __any_sync(kFull, add);
  inc_viol = __any_sync(kFull, inc_viol);
  dec_viol = __any_sync(kFull, dec_viol);
  r.cand = kInf;
  if (vmax < kInf) {  // isfinite(vmax): vmax > -inf always holds here
    double fprobe;
    if (vertical) fprobe = a.probe[side][(int64_t)cx * a.g.n + (jb + arg)];
    else fprobe = a.probe[side][(int64_t)cy * a.g.m + (ib + arg)];
    const double hc = vertical ? a.hc_x : a.hc_y;
    r.cand = vmax + 0.5 * (a.h + hc) / fprobe;  // cell_value_candidate (cells.hpp:109-112)
  }
  r.fl = 0;
  r.mon_checked = r.mon_single = false;
  if (r.add) {
    int both[2];
    mono_sides(side ^ 1, both);  // the neighbour is entered through the opposite side
    if (a.fast) {
      // sequences run north-to-south (vertical borders reversed) or west-to-east
      const bool nondec = vertical ? !dec_viol : !inc_viol;
      const bool noninc = vertical ? !inc_viol : !dec_viol;
      if (nondec && !noninc) r.fl = 1u << both[0];
      else if (noninc && !nondec) r.fl = 1u << both[1];
      else r.fl = (1u << both[0]) | (1u << both[1]);
      r.mon_checked = true;
      r.mon_single = (nondec != noninc);
    } else {
      r.fl = (1u << both[0]) | (1u << both[1]);
    }
  }
  return r;
}

__device__ __forceinline__ void hc_cell_rect(const CellGeom& g, int cell, int64_t& ib, int64_t& ie,
                                             int64_t& jb, int64_t& je) {
  const int cx = cell % g.cells_x, cy = cell / g.cells_x;
  ib = (int64_t)cx * g.base_x;
  ie = (cx == g.cells_x - 1) ? g.m : ib + g.base_x;
  jb = (int64_t)cy * g.base_y;
  je = (cy == g.cells_y - 1) ? g.n : jb + g.base_y;
}

__global__ void __launch_bounds__(32, 1) heapcell_serial_kernel(HcArgs a) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x;
  const CellGeom& g = a.g;
  HTile T;
  T.pu = g.pu;
  T.U = smem;
  T.Ct = T.U + (size_t)(g.max_h + 2) * g.pu;
  double* before = T.Ct + (size_t)(g.max_h + 2) * g.pu;  // [4][max_len]
  T.lock = reinterpret_cast<uint8_t*>(before + 4 * a.max_len);

  DevHeap H{a.hkey, a.hpos, a.harr, 0};
  if (lane == 0) {
    // cells intersecting the exit set start on the list (heap_cell.cpp:255-268)
    for (int k = 0; k < a.n_init; ++k) {
      const int cell = a.init_cells[k];
      a.cell_value[cell] = a.init_values[k];
      H.insert(cell, a.init_values[k]);
      if (a.fast) a.flags[cell] = 0xF;
    }
  }
  long long removals = 0, sweeps = 0, updates = 0, mon_checks = 0, mon_single = 0;
  for (;;) {
    int cell = -1;
    if (lane == 0 && H.size > 0) cell = H.pop();
    cell = __shfl_sync(kFull, cell, 0);
    if (cell < 0) break;
    ++removals;
    if (removals > a.budget) {  // heap_cell.cpp:276-277
      if (lane == 0) atomicExch(a.status, 3);
      break;
    }
    int64_t ib, ie, jb, je;
    hc_cell_rect(g, cell, ib, ie, jb, je);
    T.w = (int)(ie - ib);
    T.h = (int)(je - jb);
    const int cx = cell % g.cells_x, cy = cell / g.cells_x;
    // stage the cell with its cross halo (values and costs)
    const int W2 = T.w + 2;
    for (int k = lane; k < (T.h + 2) * W2; k += 32) {
      const int y = k / W2 - 1, x = k % W2 - 1;
      if ((x < 0 || x >= T.w) && (y < 0 || y >= T.h)) continue;
      const int64_t gj = jb + y;
      double v = kInf, c = -1.0;
      if (gj >= 0 && gj < g.n) {
        const int64_t o = gj * g.P + g.pad + ib + x;
        v = a.u[o];
        c = a.C[o];
      }
      T.U[(y + 1) * T.pu + (x + 1)] = v;
      T.Ct[(y + 1) * T.pu + (x + 1)] = c;
    }
    __syncwarp();
    const bool has_nb[4] = {cx > 0, cx + 1 < g.cells_x, cy > 0, cy + 1 < g.cells_y};
    // border snapshots (heap_cell.cpp:279-282)
    for (int t = lane; t < T.h; t += 32) {
      before[0 * a.max_len + t] = T.u(0, t);
      before[1 * a.max_len + t] = T.u(T.w - 1, t);
    }
    for (int t = lane; t < T.w; t += 32) {
      before[2 * a.max_len + t] = T.u(t, 0);
      before[3 * a.max_len + t] = T.u(t, T.h - 1);
    }
    unsigned my_flags = 0;
    bool first_removal = false;
    if (lane == 0) {
      my_flags = a.flags[cell];
      a.flags[cell] = 0;
      first_removal = !a.first_done[cell];
      a.first_done[cell] = 1;
    }
    my_flags = __shfl_sync(kFull, my_flags, 0);
    first_removal = __shfl_sync(kFull, (int)first_removal, 0) != 0;
    reset_locks(T, ib > 0, ie < g.m, jb > 0, je < g.n, lane);
    long long nsw = 0, upd = 0;
    if (a.fast) {
      // process_flagged_once (heap_cell.cpp:150-160)
      for (int k = 0; k < 4; ++k) {
        if (!(my_flags & (1u << kFlagOrder[k]))) continue;
        locked_sweep(T, kFlagOrder[k], lane, upd);
        ++nsw;
      }
    } else {
      // process_to_convergence (heap_cell.cpp:130-147)
      int perm[4], at = 0;
      for (int k = 0; k < 4; ++k)
        if (my_flags & (1u << kFlagOrder[k])) perm[at++] = kFlagOrder[k];
      for (int k = 0; k < 4; ++k)
        if (!(my_flags & (1u << kRotation[k]))) perm[at++] = kRotation[k];
      bool changed = true;
      while (changed) {
        const int dir = nsw < 4 ? perm[nsw] : kRotation[nsw % 4];
        changed = locked_sweep(T, dir, lane, upd);
        ++nsw;
      }
    }
    sweeps += nsw;
    for (int o = 16; o > 0; o >>= 1) upd += __shfl_xor_sync(kFull, upd, o);
    updates += upd;
    // write the cell back
    for (int k = lane; k < T.w * T.h; k += 32) {
      const int y = k / T.w, x = k % T.w;
      a.u[(jb + y) * g.P + g.pad + ib + x] = T.u(x, y);
    }
    // border scans and heap updates, sides W, E, S, N (heap_cell.cpp:288-311)
    for (int side = 0; side < 4; ++side) {
      if (!has_nb[side]) continue;
      const Scan sc = scan_side(a, T, side, before + side * a.max_len, first_removal, ib, jb, cx,
                                cy, lane);
      if (lane == 0) {
        const int nb = side == WEST ? cell - 1 : side == EAST ? cell + 1
                     : side == SOUTH ? cell - g.cells_x : cell + g.cells_x;
        if (sc.cand < a.cell_value[nb]) {
          a.cell_value[nb] = sc.cand;
          if (H.contains(nb)) H.decrease(nb, sc.cand);
        }
        if (sc.add) {
          a.flags[nb] |= (uint8_t)sc.fl;
          if (sc.mon_checked) {
            ++mon_checks;
            if (sc.mon_single) ++mon_single;
          }
          if (!H.contains(nb)) H.insert(nb, a.cell_value[nb]);
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    a.counters[0] = removals;
    a.counters[1] = sweeps;
    a.counters[2] = updates;
    a.counters[3] = mon_checks;
    a.counters[4] = mon_single;
  }
}

__global__ void heapcell_init_kernel(double* cell_value, uint8_t* flags, uint8_t* first_done,
                                     int* hpos, int J) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < J; k += gridDim.x * blockDim.x) {
    cell_value[k] = kInf;
    flags[k] = 0;
    first_done[k] = 0;
    hpos[k] = -1;
  }
}

}  // namespace

size_t heapcell_smem_bytes(const CellGeom& g, int max_len) {
  return sizeof(double) * (2 * (size_t)(g.max_h + 2) * g.pu + 4 * (size_t)max_len) +
         (size_t)g.max_w * g.max_h;
}

cudaError_t launch_heapcell(const HcArgs& args, cudaStream_t s, int* launches) {
  int blocks = (args.J + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  heapcell_init_kernel<<<blocks, 256, 0, s>>>(args.cell_value, args.flags, args.first_done,
                                              args.hpos, args.J);
  const size_t smem = heapcell_smem_bytes(args.g, args.max_len);
  cudaError_t e = cudaFuncSetAttribute(heapcell_serial_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  heapcell_serial_kernel<<<1, 32, smem, s>>>(args);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace eikb200
