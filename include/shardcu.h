/*
 * shardcu.h — C ABI of the B200 (sm_100a) dense ket engine.
 *
 * This is the drop-in boundary for the reference's hot path: the duck-typed
 * `DenseKet` class of `pkg/src/shardsim/ket.py` (bound by name at
 * engine.py:30, tableau.py:17, validate.py:20) plus the dense simulation loop
 * `dense_reference` (validate.py:83-111).  The reference has no FFI (it is
 * pure Python + NumPy), so each entry point below names the Python method it
 * replaces; the Python mirror `paper_2304_14969_b200/ket.py` binds them with
 * ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - amplitude index bit q is qubit q (qubit 0 = LSB), ket.py:3-4.
 *   - dtype SK_C64 stores float2 amplitudes, SK_C128 double2 (the reference
 *     is always complex128, ket.py:77,82).
 *   - host amplitude buffers crossing the ABI are interleaved complex128
 *     (re, im doubles) unless the function says "native".
 *   - 2x2 matrices are `const double m[8]` = re/im of m00, m01, m10, m11.
 *   - every function returns an int status; no C++ exception crosses the ABI.
 *       SK_OK 0, SK_EINDEX -> IndexError, SK_EVALUE -> ValueError,
 *       SK_ENOMEM -> DeviceMemoryError (the device is out of memory),
 *       SK_EBUDGET -> MemoryBudgetError (the engine's configured budget),
 *       SK_ECUDA -> RuntimeError.
 *     sk_last_error() returns a thread-local message for the last failure.
 *   - single writer per state (ket.py:65-66).  All work is ordered on one
 *     CUDA stream per device (sk_set_stream may replace it); functions that
 *     return host scalars synchronise that stream.
 */
#ifndef SHARDCU_H
#define SHARDCU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_OK 0
#define SK_EINDEX 1
#define SK_EVALUE 2
#define SK_ENOMEM 3
#define SK_ECUDA 4
#define SK_EBUDGET 5 /* the hybrid engine's dense-amplitude budget (engine.py:202-209) */

#define SK_C64 0
#define SK_C128 1

typedef struct sk_state sk_state;
typedef struct sk_program sk_program;

/* ---- library / device -------------------------------------------------- */
const char* sk_last_error(void);
int sk_version(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int sk_device_count(void);
/* Use `stream` (a cudaStream_t cast to an integer; 0 = the legacy default
 * stream, SK_OWN_STREAM = the library's own non-blocking stream, the
 * initial setting) for every subsequent operation on `device`. */
#define SK_OWN_STREAM UINT64_MAX
int sk_set_stream(int device, uint64_t stream);
int sk_get_stream(int device, uint64_t* stream);
int sk_synchronize(int device);
/* Free / total device memory in bytes (cudaMemGetInfo). */
int sk_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes);

/* ---- state lifetime: DenseKet.__init__ / from_amplitudes / copy ---------
 * ket.py:73-83 (|0..0> or given amplitudes), :85-91, :93-94.  width >= 1. */
int sk_create(int width, int dtype, int device, sk_state** out);
int sk_create_from(int width, int dtype, int device, const double* host_c128, sk_state** out);
int sk_copy(const sk_state* src, sk_state** out);
int sk_destroy(sk_state* s);
/* Non-owning view over caller device memory of 2^width native elements
 * (torch / NCCL buffers for the sharded path); sk_destroy frees only the
 * handle.  sk_rebind points a view at another buffer (e.g. after an
 * out-of-place all-to-all). */
int sk_wrap(int width, int dtype, int device, uint64_t ptr, sk_state** out);
int sk_rebind(sk_state* s, uint64_t ptr);
int sk_width(const sk_state* s, int* width);
int sk_dtype(const sk_state* s, int* dtype);
/* Raw device pointer of the amplitude array (for torch / NCCL plumbing). */
int sk_device_ptr(const sk_state* s, uint64_t* ptr);

/* .amps getter / setter (ket.py:82; callers engine.py:613,648,706 ...). */
int sk_upload(sk_state* s, const double* host_c128, int64_t n);
int sk_download(const sk_state* s, double* host_c128, int64_t n);
/* Same with the state's native element type (float2 or double2), for
 * pinned-buffer end-to-end copies. */
int sk_upload_native(sk_state* s, const void* host, int64_t n);
int sk_download_native(const sk_state* s, void* host, int64_t n);
/* Stream-ordered download into pinned host memory that returns without
 * waiting (the data is valid after sk_synchronize or a later synchronising
 * call on the same stream): lets a caller overlap step k's device->host
 * copy with step k+1's host->device copy and compute on another stream. */
int sk_download_native_async(const sk_state* s, void* host, int64_t n);

/* Device-to-device copies from/to a caller-owned buffer of n native
 * elements (torch / NCCL interop); stream-ordered. */
int sk_copy_from_device(sk_state* s, uint64_t src_ptr, int64_t n);
int sk_copy_to_device(const sk_state* s, uint64_t dst_ptr, int64_t n);

/* ---- gate kernels ------------------------------------------------------ */
/* DenseKet._apply_1q_unchecked (ket.py:133-144): 2x2 on pairs (i, i|2^q),
 * diagonal fast path when m01 == m10 == 0 exactly.  Unitarity is checked by
 * the caller (ket.py:57-59, 128-131). */
int sk_apply_1q(sk_state* s, int q, const double m[8]);
/* DenseKet.apply_controlled (ket.py:146-164) restricted to basis states with
 * (index & ctrl_mask) == ctrl_val.  `controls` must not contain `target`. */
int sk_apply_controlled(sk_state* s, uint64_t ctrl_mask, uint64_t ctrl_val, int target,
                        const double m[8]);
/* apply_controlled with ONE control fused with the two bloch_vector passes
 * the engine runs right after it (engine.py:389-394 -> :453): one read of
 * every amplitude; out8 = {cross_re, cross_im, n0, n1} of the control qubit
 * then of the target qubit, as sk_bloch_sums returns them. */
int sk_apply_controlled_bloch(sk_state* s, int control, int polarity, int target,
                              const double m[8], double out8[8]);
/* DenseKet.apply_pauli_layer (ket.py:166-202), in place:
 * new[j ^ flip] = old[j] * scale * (-1)^popcount(j & sign). */
int sk_apply_pauli_layer(sk_state* s, uint64_t flip, uint64_t sign, double scale_re,
                         double scale_im);
/* amps *= z (engine.py:706, tableau.py:279 "gphase"). */
int sk_scale(sk_state* s, double re, double im);
/* tableau.py _swap_bits: exchange qubits a and b (in place). */
int sk_swap_qubits(sk_state* s, int a, int b);

/* ---- reductions (fp64 accumulators, deterministic order) --------------- */
/* bloch_vector (ket.py:204-210): out4 = {Re, Im of sum conj(a0)*a1,
 * sum |a0|^2, sum |a1|^2} over the bit-q halves. */
int sk_bloch_sums(const sk_state* s, int q, double out4[4]);
/* norm (ket.py:96-97) squared. */
int sk_norm2(const sk_state* s, double* out);
/* np.vdot(a, b) (ket.py:277-281): sum conj(a)*b. */
int sk_vdot(const sk_state* a, const sk_state* b, double out2[2]);
/* amplitude(index) (ket.py:232-233). */
int sk_amplitude(const sk_state* s, int64_t index, double out2[2]);

/* ---- projections, splits, composition ---------------------------------- */
/* project_and_renormalize (ket.py:212-226): prob of `outcome` on q; if
 * prob <= 1e-12 returns SK_EVALUE leaving the state untouched; else zeroes
 * the other half and scales the kept half by 1/sqrt(prob). */
int sk_project(sk_state* s, int q, int outcome, double* prob);
/* New width-1 state holding half `half` of q scaled by (re, im):
 * out[k] = in[insert_bit(k, q, half)] * z.  Serves remove_qubit
 * (ket.py:269-275, z = 1), try_decompose's remainder (ket.py:243-267) and
 * measurement splits (engine.py:584-593). */
int sk_compact(const sk_state* s, int q, int half, double re, double im, sk_state** out);
/* Fused SDRP rounding (engine.py:464-488): out[k] = (u00*a0[k] + u01*a1[k]) * scale
 * where a0/a1 are the bit-q halves; the caller derives u and scale =
 * 1/sqrt(P0) from the Bloch sums it already holds. */
int sk_round_compact(const sk_state* s, int q, const double u0[4], double scale, sk_state** out);
/* kron_compose (ket.py:239-241): out[j * 2^wa + i] = hi[j] * lo[i]. */
int sk_kron(const sk_state* lo, const sk_state* hi, sk_state** out);
/* permute_qubits (ket.py:284-292): new qubit k is old qubit order[k]. */
int sk_permute(const sk_state* s, const int* order, sk_state** out);

/* ---- measurement -------------------------------------------------------- */
/* measure_all / sample (engine.py:596-657): numpy Generator.choice(p=|a|^2/sum)
 * is cumsum -> normalise -> searchsorted(uniforms, 'right'); the caller draws
 * the k uniforms from its own PCG64 stream, so results match draw for draw. */
int sk_sample(const sk_state* s, const double* uniforms, int64_t k, int64_t* out_idx);

/* ---- fused dense executor (validate.py:83-111's GPU analogue) ----------
 * A program is a list of sweeps; each sweep streams the state through
 * shared memory once, in tiles of 2^ntile amplitudes spanning the tile bits,
 * and applies its stages' ops on register-resident amplitudes.  See
 * DESIGN.md "Fused sweep kernel". */
#define SK_MAX_TILE_BITS 16
#define SK_MAX_REG_BITS 5
#define SK_MAX_STAGES 8

#define SK_OP_MAT 0   /* 2x2 matrix on register slot `slot`, predicated      */
#define SK_OP_DIAG 1  /* diag(d0, d1) on global qubit `qubit`, predicated     */
#define SK_OP_RAMP 2  /* phase exp(i*pi*s*F) with F = (idx >> qubit) & (2^nbits-1), predicated */
#define SK_OP_QFT 3   /* QFT layers on bits [qubit, qubit+nbits) of the window [m[0], m[1]] (each H(j)
                       * then its CP fan from all lower bits), FFT form; m[2] = previous chunk's top bit */

typedef struct {
  int32_t kind;
  int32_t qubit;     /* MAT: target qubit; DIAG: qubit; RAMP: field low bit */
  int32_t nbits;     /* RAMP: field width (<= 62) */
  int32_t pad;
  uint64_t ctrl_mask;
  uint64_t ctrl_val;
  double m[8];       /* MAT: 2x2; DIAG: d0 = m[0..1], d1 = m[6..7]; RAMP: s = m[0] */
} sk_op;

typedef struct {
  int32_t ntile;                              /* tile bits T */
  int32_t tile_bits[SK_MAX_TILE_BITS];        /* ascending global bit positions */
  int32_t nstages;
  int32_t reg_bits[SK_MAX_STAGES][SK_MAX_REG_BITS]; /* global qubits held in registers */
  int32_t op_begin[SK_MAX_STAGES + 1];        /* stage s runs ops[op_begin[s] .. op_begin[s+1]) */
  int32_t nreg;                               /* register bits per stage: 0 = sk_program_reg_bits default;
                                                 c64: 4 (5 for QFT-window sweeps), c128: 3 or 4 */
} sk_sweep;

/* Validate and upload a program for an n-qubit state of `dtype`.  Each
 * sweep's `nreg` is the register-bit count it was planned with
 * (sk_program_reg_bits gives the dtype default).  A sweep whose lowered ops
 * all have fast paths and number at most 128 runs with its op table in the
 * kernel's parameter space (k_sweep LEAN); longer or more general sweeps run
 * through the op interpreter — same results, slower. */
int sk_program_reg_bits(int dtype, int* nreg);
int sk_program_create(int width, int dtype, int device, const sk_sweep* sweeps, int nsweeps,
                      const sk_op* ops, int nops, sk_program** out);
int sk_program_destroy(sk_program* p);
/* Host-only introspection (no device needed): lower a program into the
 * fused kernel's op list.  For each kernel op i: ints[12i..12i+11] =
 * {kind, slot, pattern, element mask, flags, lo, nbits, tmask, tval, qmask,
 * turn, field mask}, reals[24i..24i+23] = coefficients m[8] then twiddles tw[16].  stage_ops[(SK_MAX_STAGES+1)*s + t]
 * = first kernel op of stage t of sweep s (the entry after the last stage
 * holds the end).  Used by the CPU tests to emulate the kernel ops. */
int sk_program_lower(int width, int dtype, const sk_sweep* sweeps, int nsweeps, const sk_op* ops, int nops,
                     int64_t* ints, double* reals, int cap, int* count, int* stage_ops);
/* Run sweeps [first, first+count) of the program on s (count < 0: all). */
int sk_program_run(sk_state* s, const sk_program* p, int first, int count);
int sk_program_nsweeps(const sk_program* p, int* n);
/* Sharded QFT (no reference counterpart): run a QFT-window
 * program planned for an (n-G)-qubit shard as the top n-G layers of an
 * n-qubit QFT whose low G qubits are fixed to `value` on this rank (their
 * controlled phases fold into the windows' twiddles).  shift = G; 0 clears. */
int sk_program_set_phase_index(sk_program* p, int shift, uint64_t value);
/* Run tiles [tile_begin, tile_end) of one QFT-window sweep (the exchange
 * overlap of the sharded QFT launches its last body sweep block by block, so
 * each finished block's transfer starts while the next block computes). */
int sk_program_run_tiles(sk_state* s, const sk_program* p, int sweep, int64_t tile_begin, int64_t tile_end);
/* Tile geometry of a sweep: *tile_bits = T (negated when the tiles are not
 * contiguous index ranges), *tiles = 2^(width - T). */
int sk_program_sweep_tiles(const sk_program* p, int sweep, int* tile_bits, int64_t* tiles);

/* ---- native hybrid engine (engine.py HybridState, dense shards) ---------
 * The factorised simulator's commit stream runs in C++ next to the kernels:
 * 1q buffers, pending controlled-op queues, control elimination, merges,
 * exact splits and SDRP rounding with the reference's rules
 * (engine.py:164-784 with OptFlags(stabilizer_hybrid=False)); the decision
 * inputs come back from the device through mapped pinned memory.  Gates are
 * passed as packed arrays; matrices are the gate_matrix() values. */
typedef struct sk_engine sk_engine;

typedef struct {
  double sdrp;             /* EngineConfig.sdrp in [0, 1] (engine.py:66-78) */
  double separability_tol; /* 1e-10 */
  int64_t mem_budget;      /* dense amplitudes */
  int32_t dtype;           /* SK_C64 / SK_C128 */
  int32_t device;
  int32_t control_elimination, hx_commutation, label_swap, pauli_coalescing; /* OptFlags */
  int32_t stabilizer_hybrid; /* OptFlags.stabilizer_hybrid: qubits start as width-1 tableaus (tableau.py) */
} sk_engine_config;

#define SK_GATE_1Q 0      /* 2x2 on targets[2g] (with controls when ctrl_off[g+1] > ctrl_off[g]) */
#define SK_GATE_SWAP 1    /* targets[2g], targets[2g+1] */
#define SK_GATE_MEASURE 2 /* targets[2g]; draws one uniform from the engine's rng callback */

#define SK_ENGINE_STAT_LABEL_SWAPS 0
#define SK_ENGINE_STAT_KERNELS 1
#define SK_ENGINE_STAT_ELIMINATED 2
#define SK_ENGINE_STAT_MERGES 3
#define SK_ENGINE_STAT_SPLITS 4
#define SK_ENGINE_STAT_ALLOCS 5      /* device states created (ket.py alloc_count) */
#define SK_ENGINE_STAT_WRITES 6      /* amplitudes written (ket.py amplitude_writes) */
#define SK_ENGINE_STAT_DENSE_TOTAL 7
#define SK_ENGINE_STAT_PEAK 8        /* peak_amplitudes */
#define SK_ENGINE_STAT_NEPS 9        /* len(eps_record) */
#define SK_ENGINE_STAT_NEEDED 10     /* `needed` of the last SK_EBUDGET */
#define SK_ENGINE_STAT_DIST_SHARDS 11 /* shards split over the ranks (sk_engine_set_distributed) */
#define SK_ENGINE_STAT_EXCHANGES 12  /* rank-bit <-> slab-bit swaps of distributed shards */
#define SK_ENGINE_NSTATS 13

typedef double (*sk_uniform_fn)(void* ctx); /* rng.random() of the caller's PCG64 stream */
typedef int (*sk_bit_fn)(void* ctx);        /* rng.integers(0, 2) of the same stream (tableau measurements) */
/* collectives of the distributed largest shard, provided by the host's
 * process group (torch.distributed: NCCL on the box, gloo in the tests);
 * each returns 0 on success and completes before returning */
typedef int (*sk_allreduce_fn)(void* ctx, double* x, int n); /* in-place sum over ranks of n host doubles */
typedef int (*sk_sendrecv_fn)(void* ctx, int partner, uint64_t send_dev, uint64_t recv_dev, int64_t nbytes);
typedef int (*sk_allgather_fn)(void* ctx, uint64_t send_dev, uint64_t recv_dev, int64_t nbytes_per_rank);

/* HybridState(n, cfg) (engine.py:164-182): n width-1 shards |0>. */
int sk_engine_create(int n, const sk_engine_config* cfg, sk_engine** out);
int sk_engine_destroy(sk_engine* e);
int sk_engine_set_rng(sk_engine* e, sk_uniform_fn fn, void* ctx);
int sk_engine_set_rng_bits(sk_engine* e, sk_bit_fn fn, void* ctx);
/* SPMD distribution: every rank runs the same engine on the
 * same circuit; a dense shard wider than local_max_width is split over the
 * `world` ranks by its top log2(world) positions (merges with replicated
 * shards grow every slab locally; gates, Bloch sums and SDRP rounding act on
 * local positions, rank-bit qubits are swapped into the slab by pairwise
 * exchanges; reductions are summed over ranks, so every rank takes the same
 * decisions) and gathered back once it narrows to local_max_width. */
int sk_engine_set_distributed(sk_engine* e, int world, int rank, int local_max_width, sk_allreduce_fn allreduce,
                              sk_sendrecv_fn sendrecv, sk_allgather_fn allgather, void* ctx);
/* apply_gate for gates [0, ngates) (engine.py:514-573): kind[g], targets[2g..2g+1],
 * controls ctrls[ctrl_off[g] .. ctrl_off[g+1]) with polarities pols[...], matrix mats[8g..8g+7].
 * *done = gates fully applied (the failing gate is not counted). */
int sk_engine_apply(sk_engine* e, int ngates, const int32_t* kind, const int32_t* targets, const int32_t* ctrl_off,
                    const int32_t* ctrls, const int32_t* pols, const double* mats, int* done);
/* _measure_qubit (engine.py:575-594). */
int sk_engine_measure(sk_engine* e, int label, int* outcome);
/* flush_all (engine.py:669-681) / flush_buffers(q). */
int sk_engine_flush_all(sk_engine* e);
int sk_engine_flush_qubit(sk_engine* e, int label);
/* sdrp_round(q, p) (engine.py:490-512): *eps_out = recorded eps or -1. */
int sk_engine_sdrp_round(sk_engine* e, int label, double p, double* eps_out);
int sk_engine_stats(const sk_engine* e, int64_t out[SK_ENGINE_NSTATS]);
int sk_engine_eps(const sk_engine* e, double* out, int64_t cap);
/* The shards in label order (engine.py _shards_in_label_order): states[i]
 * (borrowed handles valid until the next engine call; owned[i] = 1 for a
 * tableau shard's freshly replayed dense ket, which the caller destroys),
 * widths[i], and each shard's qubit labels by position, shard after shard. */
int sk_engine_shards(sk_engine* e, int cap, sk_state** states, int* widths, int* labels, int* owned, int* nshards);
/* load_state (engine.py:768-784): one dense shard, label i = bit i. */
int sk_engine_load_state(sk_engine* e, const sk_state* s);
/* measure_all (engine.py:596-626): bits[label] = outcome, dense shards
 * collapse to fresh width-1 shards, tableaus in place. */
int sk_engine_measure_all(sk_engine* e, uint8_t* bits);
/* sample(shots) without collapse (engine.py:628-657): bits[shot * n + label]. */
int sk_engine_sample(sk_engine* e, int64_t shots, uint8_t* bits);

#ifdef __cplusplus
}
#endif
#endif /* SHARDCU_H */
