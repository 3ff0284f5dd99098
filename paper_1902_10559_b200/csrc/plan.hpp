// SART plan: the device-resident iteration loop of reference sart_solve
// (proj/src/solvers.cpp:148-199) over one system or the folded pair.
#pragma once

#include "internal.hpp"

namespace ssb {

// Fused row-sharded exchange over peer memory (replaces the NCCL all-reduce of
// the back-projection; sart.cu "peer exchange"). Every rank owns one region
// (plain cudaMalloc, IPC-exportable) with the same layout:
//   recv [G][cols]  row g: rank g's partial back-projection of the columns
//                   this rank owns ([me*own, (me+1)*own))
//   x    [cols]     this rank's replica of the iterate
//   r2   [2][G]     ||r_g||^2 of every rank, by iteration parity
//   done            ranks whose K2x finished (monotone over solves)
//   xready          owners whose reduce pushed their x range here
//   dflag           first diverged iteration (+1) seen by any owner
struct PeerExchange {
  int G = 1, me = 0;
  bool emulated = false;  // all ranks' plans on one device, launched in rank order
  std::int64_t cols = 0, own = 0;  // columns, columns owned per rank
  int rgrid = 0;                    // CTAs of the reduce kernel
  std::size_t off_recv = 0, off_x = 0, off_r2 = 0, off_done = 0, off_xready = 0,
              off_dflag = 0, bytes = 0;
  void* region = nullptr;
  std::vector<void*> opened;  // peers' regions mapped through CUDA IPC
  DBuf<char*> peers;          // [G] region base of every rank as seen from this device
  DBuf<long long> local;      // {epoch base, iterations proceeded, timeout, reduces announced}
  ~PeerExchange();
};

struct Plan {
  Context* ctx = nullptr;
  int nsys = 1;
  int nrhs = 1;
  int dtype = SS_F64;
  int vs_fwd = 32, vs_back = 8;
  int uf_fwd = 2, uf_back = 2;  // load steps in flight per lane before the gathers
  int fwd_blocks = 0, back_blocks = 0;
  bool sharded = false;
  bool paired = false;  // folded pair on one shared index stream
  Matrix* pair_own[2] = {nullptr, nullptr};  // union-pattern copies (when patterns differ)
  int sys_blocks_f = 0x7fffffff, sys_blocks_b = 0x7fffffff;  // first CTA of system 1
  std::int64_t row_begin = 0, row_end = 0;  // sharded: rows kept by this rank
  ss_solve_options opts{};
  Matrix* a[2] = {nullptr, nullptr};
  // Row-sharded plans own a row-block copy of the (single) system.
  Matrix* own = nullptr;
  Matrix* own2 = nullptr;  // row-sharded pair: the local block of A2
  std::int64_t rows[2] = {0, 0}, cols[2] = {0, 0};
  // per system, plan dtype (T) buffers in bytes
  DBuf<char> x[2], w[2], p[2], rinv[2], cinv[2];
  DBuf<double> partial;   // [nsys*nrhs][fwd_blocks]
  DBuf<double> pnorm;     // [nsys*nrhs]
  DBuf<double> history;   // [nsys*nrhs][max_iters+1]
  DBuf<int> state;        // [nsys*nrhs][4] stopped, stop_it, diverged_at, -
  DBuf<unsigned> ticket;  // last-block ticket of the forward kernel
  DBuf<char> bp;          // sharded: back-projection + ||r||^2 slot (all-reduced)
  PeerExchange* px = nullptr;  // sharded over peer memory instead of NCCL
  DBuf<char> xx, ww;      // paired: interleaved x [cols][2] and w [rows][2]
  DBuf<char> rv2, cv2;    // paired: CSR / CSC values interleaved [nnz][2]
  DBuf<char> pe, cc;      // paired: {p1,p2,rinv1,rinv2} per row, {cinv1,cinv2} per column
  // multi-RHS block-merged streams (sart_*_block_kernel): per direction the
  // union list of every block of kBlockR vectors over both folded systems
  bool blocked_f = false, blocked_b = false;
  int block_e_f = 4, block_e_b = 2;  // union entries' gathers in flight per lane
  DBuf<int> bptr_f, bidx_f, bptr_b, bidx_b;
  DBuf<char> bval_f, bval_b;
  std::int64_t nblk_f = 0, nblk_b = 0, nu_f = 0, nu_b = 0;
  // multi-RHS K1 / K2 with the gathered operand staged through a bulk-copy
  // ring (sart_stage_kernel): per direction, per block of kStageR vectors of
  // each system its index union and its entries chunk-major (row / column
  // pairs merged) with their position in the chunk
  struct StageBufs {
    bool on = false;
    DBuf<int> bptr, buni, bch;
    DBuf<long long> cofs;
    DBuf<char> ent;
    std::int64_t nblk = 0, nu = 0, entb = 0;
    int slot = 0, smem = 0, blocks = 0;
  } stg[2];  // [0] K1 (rows, X), [1] K2 (columns, W)
  int nband = 1;          // multi-RHS K1 passes over column bands
  DBuf<int> band_ptr[2];  // per system [nband + 1][rows] positions inside the CSR rows
  // paired + tiled: rows/columns padded to 4 entries and permuted within tiles
  // of 4*VS entries so each gather instruction covers consecutive entries
  bool tiled = false;
  // tiled + 16-bit indices: per tile an int32 base, per entry a uint16 offset
  bool c16f = false, c16b = false;  // per direction (K1 rows / K2 columns)
  DBuf<unsigned short> tofs_f, tofs_b;
  DBuf<int> tbase_f, tbase_b, tfirst_f, tfirst_b;  // per tile base, per vector first tile
  std::int64_t ntile_f = 0, ntile_b = 0;
  // tiled + 16-bit + mirror-coded pair values (see seg_dot2m): per tile header
  // {base, sign words} (hs words), one value per entry, exception lists
  bool mir_f = false, mir_b = false;
  int hs_f = 0, hs_b = 0;
  DBuf<unsigned> thdr_f, thdr_b;
  DBuf<int> eptr_f, eptr_b, eidx_f, eidx_b;
  DBuf<char> ev2_f, ev2_b;
  std::int64_t nexc_f = 0, nexc_b = 0;
  bool stream_cs = false;  // evict-first hint on the stream loads (fp32, stream > L2)
  bool l2_window = false;  // persisting L2 access-policy window on the gathered vector
  int layout_mode(bool fwd) const {
    if (!tiled) return 0;
    if (!(fwd ? c16f : c16b)) return (fwd ? mir_f : mir_b) ? 6 : 1;
    if (fwd ? mir_f : mir_b) return stream_cs ? 5 : 4;
    return stream_cs ? 3 : 2;
  }
  // persistent loop (sart_persistent_pair_kernel): one cooperative launch per
  // solve, grid barriers between the K1 and K2 phases
  bool persistent = false;
  int pgrid = 0;
  // stream-resident persistent loop (sart_resident_pair_kernel): one CTA per
  // SM, both streams staged in shared memory once per launch (csmem bytes)
  bool resident = false;
  bool res_back = true;  // K2's stream staged too (false: only K1's fits)
  // cluster-persistent loop (sart_cluster_pair_kernel): the grid is one
  // thread-block cluster of ccluster CTAs, hardware cluster barriers
  bool cluster = false;
  int ccluster = 0;
  int csmem = 0;  // its dynamic shared memory per CTA (staged streams)
  DBuf<unsigned> gbar;  // {arrivals, generation}
  DBuf<int> tptr_f, tptr_b, tidx_f, tidx_b;
  std::int64_t tnnz_f = 0, tnnz_b = 0;
  cudaGraphExec_t graph = nullptr;
  cudaGraphConditionalHandle cond = 0;  // WHILE node of the captured loop
  DBuf<int> iter_dev;                     // pass counter of the captured loop
  bool while_capture = false;             // make_args: kernels read / advance iter_dev
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  float last_ms = 0.0f;
  float group_ms = -1.0f;
  double pn_local[2] = {-1.0, -1.0};  // emulated exchange rank: local ||p_g|| (run_group combines)  // emulated exchange group: time of the whole group's solve
  bool launched = false;
  bool empty_rows[2] = {false, false};  // all row sums zero (reference throws)

  ~Plan();
  std::size_t tsize() const { return dtype == SS_F32 ? 4 : 8; }
  void build_graph();
  void enqueue_iterations(int first, int count);  // raw launches (no graph)
  void enqueue_reset();
  void enqueue_epilogue();  // paired: de-interleave x1/x2
  void set_rhs_host(int which, const double* p_slice_major);
  void set_rhs_device(int which, const void* p_dev);
  void set_rhs_device_f64(int which, const double* p_dev);  // [rows] fp64, nrhs == 1
  void finish_rhs(int which);  // ||p|| (all-reduced for sharded plans)
  int diverged_at(int which) const;
  void recombine_device(double* f_dev);  // N = 2*cols fp64, nrhs == 1
  void launch();
  void finish(ss_solve_report* rep);
  void get_solution(int which, double* f_slice_major);
  void get_history(int which, int slice, double* h, int* len);
  void recombine(double* f_slice_major);
  void profile(int iters, float* fwd_ms, float* back_ms);
  void time_kernel(bool fwd, int reps, float* ms);
  void stats(std::int64_t* mbytes, std::int64_t* vbytes, int* kernels) const;
  void kernel_bytes(std::int64_t* fwd, std::int64_t* back) const;
  std::string describe() const;
};

Plan* make_plan(Context* ctx, Matrix* a1, Matrix* a2, const ss_solve_options& o, int nrhs,
                bool reusable = true);
// exchange: SS_XCHG_NCCL or SS_XCHG_PEER. emul_parts > 0 builds rank
// emul_rank of a one-device emulation (no communicator; see run_group).
// The folded pair row-sharded over all ranks (peer exchange, paired streams);
// emul_parts > 0: rank emul_rank of a one-device emulation.
Plan* make_sharded_pair_plan(Context* ctx, Matrix* a1, Matrix* a2, std::int64_t row_begin,
                             std::int64_t row_end, const ss_solve_options& o, int emul_parts = 0,
                             int emul_rank = 0);
Plan* make_sharded_plan(Context* ctx, Matrix* a, std::int64_t row_begin, std::int64_t row_end,
                        const ss_solve_options& o, int exchange = SS_XCHG_NCCL,
                        int emul_parts = 0, int emul_rank = 0);
// link the plans of a one-device emulation to each other's exchange regions
void link_group(Plan* const* plans, int parts);
// one solve of an emulated group: all ranks' launches in rank order on the
// shared stream (no launch ever waits on one that has not completed)
void run_group(Plan* const* plans, int parts);
void partition_rows(const int* rowptr, std::int64_t rows, int parts, std::int64_t* bounds);
void exchange_owned_columns(std::int64_t cols, int parts, int rank, std::int64_t* begin,
                            std::int64_t* end);

}  // namespace ssb
