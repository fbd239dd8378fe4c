// Internal interface between the host runtime (eik_abi.cpp) and the kernels.
#pragma once

#include <cstdint>
#include <cuda.h>  // CUtensorMap (the FMSM tile loads)
#include <cuda_runtime.h>

namespace eikb200 {

// Device layout of every plan (chosen for the kernels, not the caller):
// value field u and cost C = h/F are stored with a row pitch P = m + 2*kPad
// and rows -1..n (the base pointer is row 0); grid node (i,j) lives at
// j*P + kPad + i.  Padding columns and
// the dummy row n hold u = +inf, C = -1 (the exit/no-update marker), so the
// sweep kernels never test bounds.
constexpr int64_t kPad = 64;

struct FsmArgs {
  const double* C;          // padded h/F, -1 for exits and padding
  double* u;                // padded value field
  int64_t m, n, P, pad;
  int nstrips;              // ceil(n / 32)
  unsigned long long* prog; // [nstrips] sweeps completed by each strip
  double* mbox;             // [2][nstrips] rows of pitch P: edge-row mailboxes
  int* changed;             // [max_sweeps] change flag per sweep
  int* done;                // [max_sweeps] strips finished per sweep
  int max_sweeps;
  int lookahead;            // D: stop decision for sweep k uses sweep k-D
  int first_sweep;          // direction of local sweep k is (first_sweep + k) mod 4
  int fixed;                // run exactly max_sweeps sweeps (no stop decision)
  int* status;              // [0] error, [1] sweeps
  unsigned long long* trace; // optional [kTraceSweeps][nstrips][kTraceWords]: globaltimer
                             // (start, body start, end), polls, compute steps
  // Change bits (k_fsm.cu): [2][n+3][cw] u32, bit i of row r in sweep parity
  // k&1 = node (i,r) decreased in sweep k.  Row r at (r+1)*cw, column word w
  // at +w+kChgWordOff; the pad rows/words are never written (stay zero).
  unsigned* chg;
  int64_t cw;               // words per row: ceil(m/32) + kChgWordPad
  int noskip;               // evaluate every node (no clean-step skipping)
  // Strip-Jacobi partitions (0: one Gauss-Seidel wavefront over all rows):
  // parts of part_strips strips sweep side by side, reading the neighbouring
  // part's edge row as it was at the end of the previous sweep from
  // snap[k&1][boundary][side][P] (side 0: the lower part's top row, side 1:
  // the upper part's bottom row; padded rows, +inf before the first sweep).
  int part_strips;
  double* snap;
  // LSM (lsm_solve, classic_solvers.cpp:160-212): when non-null, the sweep
  // also counts the nodes the reference's locking sweep processes
  // (lsm_cnt[k] += unlocked nodes of sweep k).  Values and sweeps are FSM's.
  unsigned long long* lsm_cnt;
  // Super-block skipping (k_fsm.cu): a strip's sweep is cut into super-blocks
  // of kFsmSbBlocks blocks; sb holds [2][nstrips][nsb] per-sweep-parity update
  // summaries (bit 0 any row, bit 1 the strip's lowest row, bit 2 its highest)
  // followed by [2][nstrips][nsb] edge tokens per row direction (sweep stamp
  // << 2 | state; zeroed before every launch).  Null: no super-block skipping.
  unsigned* sb;             // ... then [nstrips] steps each strip computed in its last sweep
  int nsb;
  int cont;                 // continuing launch: sweep 0 uses the change bits its predecessor left
  int par0;                 // parity offset: sweep k writes parity (k + par0) & 1
  int start_ahead;          // a computed run starts once the upwind strip is this many columns ahead
  int sb_wait_div;          // a strip waits for upwind tokens when it computed fewer than
                            // (m + 31) / sb_wait_div steps in its previous sweep (0: never)
};
constexpr int kFsmSbBlocks = 4;    // blocks of 8 steps per super-block (32 steps; 16 and 128 measured slower)
constexpr int kFsmSbMaxPerRow = 4096;  // the kernel's shared-memory dirty map (k_fsm.cu kMapWords)
inline int fsm_nsb(int64_t m) {
  const int64_t nblocks = (m + 31 + 7) / 8;
  return (int)((nblocks + kFsmSbBlocks - 1) / kFsmSbBlocks);
}
constexpr int64_t kChgWordOff = 3;
constexpr int64_t kChgWordPad = 8;  // pad words per row (kChgWordOff before, the rest after)
constexpr int kTraceSweeps = 16;
constexpr int kTraceWords = 8;  // start, body start, end, polls, compute steps, skipped super-blocks,
                                // ns and blocks in computed runs

// Cell decomposition as seen by the device (build_cells, cells.cpp:32-47):
// cell (cx,cy) spans columns [cx*base_x, cx==cells_x-1 ? m : (cx+1)*base_x).
struct CellGeom {
  int64_t m, n, P, pad;
  int cells_x, cells_y;
  int64_t base_x, base_y;
  int max_w, max_h;         // largest cell (the last row/column of cells)
  int pu, pc;               // even smem pitches of the u tile (w+2) and C tile (w)
  int64_t row0, row_end;    // node rows of cell row 0 / end of the last cell row
                            // (0 and n, except on a sharded FMSM's strip)
  int64_t tile_doubles;     // per-warp smem: (max_h+2)*pu + max_h*pc
};

struct FmsmArgs {
  CellGeom g;
  const double* C;          // padded h/F
  double* u;                // padded values
  const int32_t* order;     // cells in coarse order
  const int32_t* rank;
  const uint8_t* flags;     // bit d: sweep direction d chosen; bit 4: Q-cell
  int* done;                // [J] cell finished
  int* next;                // claim counter
  unsigned long long* counters;  // [0] sweeps, [1] node updates
  int* status;
  int J;
  int max_cell_sweeps;
  int big;                  // cells too large for a shared-memory tile: swept in place
  // Tile staging by TMA: 2-D tensor maps over the padded u / C from row -1
  // (pitch P), box pu x (max_h + 2) = one tile with its halo; the cost tile
  // sits tile_doubles / 2 after the value tile (both 128-byte aligned)
  int use_tma;
  const CUtensorMap* tmaps;  // device memory: [0] u, [1] C
  int nowait;               // a level of a sharded solve: the listed cells are
                            // pairwise non-adjacent and their inputs final
};

// max_ctas caps the persistent grid (0: the whole device) so that plans can
// share a GPU (eik_plan_run_batch); *_capacity report the CTAs the whole
// device holds for that kernel configuration.
cudaError_t launch_fmsm(const FmsmArgs& a, int warps_per_cta, int max_ctas, cudaStream_t s,
                        int* launches, int* grid = nullptr);
cudaError_t fmsm_capacity(int64_t tile_doubles, int warps_per_cta, int* ctas);

// Result of processing one cell (sweeps + the four border scans): the
// per-warp staging copy in shared memory that process_cell fills.
struct alignas(16) SpecRec {
  double cand[4];
  int sweeps, updates;
  unsigned inst;            // instance number
  unsigned tag;             // version of the cell the result is valid at
  unsigned side[4];         // per side: bit 0 add, bits 8-15 sweep flags, bit 16
                            // monotonicity checked, bit 24 single-direction
  unsigned dmask;           // chained: sides whose pending results it assumes
  unsigned dinst[4];        // ... and their instance numbers
  unsigned nseq;            // unused in the staging copy
};

// The published speculation record in global memory: eight 16-byte words,
// each written and read as ONE single-copy-atomic 128-bit access (PTX
// ld/st .b128).  Every word carries the instance number of the write it
// belongs to, so a reader that loads the words it needs in one batch -- no
// ordering between the loads -- knows they come from one complete write iff
// their instance numbers agree.
//   word d (0-3): cand[d] (f64 bits) | side[d] | inst
//   word 4:       sweeps | updates | tag | inst
//   word 5:       dmask | dinst[0] | dinst[1] | inst
//   word 6:       dinst[2] | dinst[3] | nseq (writes so far) | inst
struct alignas(128) PRec {
  uint4 w[8];
};

struct HcArgs {
  CellGeom g;
  double* slots;            // [3][J][max_h*max_w] per-cell value slots
  int64_t cellsz;           // max_h * spw
  int spw;                  // slot row pitch: max_w rounded up to even
  unsigned long long* state;  // [J] packed state word (k_heapcell.cu)
  unsigned* spec_ver;       // [2][J] tag of the plain / chained speculation
  int* busy;                // [2][J] a warp is computing that speculation
  PRec* rec;                // [2][J] published speculation records
  int use_tma;              // tiles by TMA: the replay's cost tiles (tmc: the padded
  const CUtensorMap* tmc;   // C from row -1), the band rounds' value and cost
  const CUtensorMap* tm_band;  // tiles (tm_band: [u, C])
  double* ckey;             // [J] heap key published for the workers (inf = not queued)
  unsigned* ctag;           // [J] instance number of the last committed result
  int chain;                // make chained speculations
  int bands;                // cells of 33-128 rows swept as 32-row bands (k_cellsweep.cuh)
  int idle_ns;              // worker back-off when it found nothing to do
  int prof;                 // run the instrumented kernel (EIK_HC_PROFILE)
  int* wdbg;                // optional debug: [workers][4] phase, cell, kind, time
  int* owner;               // optional debug: [2][J] last claiming worker
  int* done_flag;
  int* hsize_pub;           // per-bucket queue counts for the workers, bucket b at [32 b]
  int* pubmin;              // per-bucket minimum id for the workers (-1 empty), [32 b]
  int first_min;            // workers wid < 32 * first_min try their bucket's minimum first ...
  int first_min_pool;       // ... in pools of at most this many workers
  int64_t tile_doubles;     // per-warp smem
  int64_t min_smem;         // launch at least this much dynamic smem per CTA (SM-exclusive CTAs)
  unsigned long long cx_magic;
  int skip_from;            // HCM: sweeps from this one on use the vote-skip engine  // cell / cells_x == (cell * cx_magic) >> 40 for every cell (0: divide)
  int heap_cap;             // >0: committer queue buckets in shared memory, capacity
                            // per bucket; 0: buckets in global memory (hkey + harr)
  int heap_capb_global;     // bucket capacity of the global layout (ceil(J/32))
  int pub_capb;             // bucket stride of the published id mirror (harr)
  const double* C;          // padded h/F
  double* u;                // padded values
  const double* probe[4];   // F at border probe points: W/E [cells_x*n], S/N [cells_y*m]
  double h, hc_x, hc_y;
  double* cval;             // [J] cell values (heap_cell.cpp cell_value)
  double* hkey;             // [32][capb] queue keys (global-bucket mode)
  int* hpos;                // [J] queue position of every cell (bucket << 24 | slot), -1
  int* harr;                // [32][capb] queue ids: mirror for the workers / global buckets
  const int* init_cells;    // Q-cells in ascending id order with their initial values
  const double* init_values;
  int n_init;
  unsigned long long* counters;  // removals, sweeps, node updates, mon checks, mon single
  int* status;
  int J;
  int fast;                 // 0 = HCM, 1 = FHCM
  long long budget;         // removal budget 100*J+16 (heap_cell.cpp:270)
  int max_len;              // longest cell side
  // HCM band scheduler (hcm_band_kernel): rounds of mutually non-adjacent
  // queued cells within the acceptance band [kmin, kmin + delta]
  int* b_inq;               // [J] cell is queued
  unsigned* b_flags;        // [J] raised sweep flags
  unsigned char* b_fdone;   // [J] first removal done
  int* b_list;              // [2][J] queued cells (ping-pong by round parity)
  int* b_work;              // [J] cells selected this round
  int* b_ctl;               // [0..1] list sizes, [2] selected count, [3] dispenser, [4] rounds
  unsigned long long* b_kmin;  // [0] round minimum key bits, [1] minimum C bits
  double band_scale;        // delta = band_scale * (h + min(hc_x, hc_y)) / (2 F_max)
  int band_adapt;           // widen / narrow the band by the cells a round selects
  int band_shrink;          // ... narrowing after a round of more cells than this
  // cells too large for a shared-memory tile (heapcell_serial_kernel): the
  // exact heap loop, one warp, cells swept in place in u
  uint8_t* big_lock;        // [max_h * max_w] lock bytes
  double* big_scratch;      // [8 * max_len] border snapshots + probe strips
};

size_t heapcell_smem_bytes(const CellGeom& g, int max_len);
size_t heapcell_committer_heap_bytes(int cap);
cudaError_t launch_heapcell(const HcArgs& a, int warps_per_cta, int max_ctas, cudaStream_t s,
                            int* launches, int* grid = nullptr);
cudaError_t heapcell_capacity(int64_t tile_doubles, int heap_cap, int warps_per_cta,
                              size_t min_smem, int* ctas);
cudaError_t launch_hcm_band(const HcArgs& a, int warps_per_cta, int max_ctas, cudaStream_t s,
                            int* launches, int* grid = nullptr);
cudaError_t launch_heapcell_serial(const HcArgs& a, cudaStream_t s, int* launches);
cudaError_t hcm_band_capacity(int64_t tile_doubles, int warps_per_cta, size_t min_smem,
                              int* ctas);
// Raise a kernel's dynamic shared-memory limit to at least `bytes` (never
// lowers it: concurrent launches of the same kernel from other host threads
// may need the larger limit).
cudaError_t ensure_dynamic_smem(const void* kernel, size_t bytes);

cudaError_t launch_prepare(const double* F, double* C, double* u, int64_t m, int64_t n,
                           int64_t P, int64_t pad, double h, const int64_t* exits,
                           const double* cost, int64_t n_exit, int* status, cudaStream_t s,
                           int* launches);
cudaError_t launch_fsm(const FsmArgs& a, cudaStream_t s, int* launches, int* grid = nullptr);
cudaError_t launch_set_rows_marked(double* u, const double* src, int64_t row0, int64_t nrows,
                                   int64_t m, int64_t P, int64_t pad, unsigned* chg_par, int64_t cw,
                                   unsigned* sum_par, int nsb, cudaStream_t s);
cudaError_t launch_fill(double* p, int64_t count, double v, cudaStream_t s, int* launches);
cudaError_t fsm_capacity(int nstrips, int* need, int* ctas, bool lsm = false);

cudaError_t device_acceptance_order(const double* u, const double* C, int64_t m, int64_t n,
                                    int64_t P, int64_t pad, int32_t* order_dev, cudaStream_t s);
cudaError_t pool_alloc(void** p, size_t bytes);
void pool_release(void* p);

cudaError_t device_metrics(const double* vm, const double* ve, const double* vt, int64_t M,
                           const int64_t* exits, int64_t n_exit, uint8_t* mask, cudaStream_t s,
                           double res[5], long long counts[2]);

}  // namespace eikb200
