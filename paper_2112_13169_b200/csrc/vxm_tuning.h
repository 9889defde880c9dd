// Build-time tuning knobs of the kernels and the runtime, in one place. The
// defaults are the measured optima on B200 (tools/ab_build.sh builds a
// variant library with -D overrides; tools/quick_time.py / bench.py time it
// with VXM_LIB_NAME=...). Product code never tests these names anywhere else.
#pragma once

// FrameParams device buffers (each with its own instance of every frame
// graph): the upload for call k+1 runs while call k's graph executes. 3 and 4
// measured no faster than 2.
#ifndef VXM_PP
#define VXM_PP 2
#endif

// Graph branches of a batch (equal shares of the streams, desynchronised
// per-branch graphs): 3 beat 2, 4 and 6 (64 cfg2 streams: 2 branches -9%,
// 4 branches -3%).
#ifndef VXM_BRANCHES
#define VXM_BRANCHES 3
#endif

// Batch ray-cast shape: kChunk steps per resolve, warps per block, resident
// blocks per SM (which sets the register cap: 20 x 2 warps -> 48 registers),
// fast (threshold-free) chunks. Measured alternatives, 64 cfg2 streams:
// chunk 8 -25% frames/s, 4-warp blocks at 40 registers -1%. Round 2: with
// the per-axis fast-chunk bound, fma steps and live-lane resolves, fast
// chunks are +5% (K3 146 -> 136 us per step) and 20 blocks (48 registers,
// no spills) +0.5% over 24 (40 registers); before them fast chunks were -4%
// and 20 blocks -2%.
#ifndef VXM_TB_CHUNK
#define VXM_TB_CHUNK 4
#endif
#ifndef VXM_TB_WARPS
#define VXM_TB_WARPS 2
#endif
// K3 (one-warp kernel of lone frames / small calls): fast chunks in the warp's
// tail with the ended lanes masked (1) or exact chunks from the first ended
// lane on (0). r02ch: lone cfg2 27.8 -> 27.2 us, cfg1 26.2 -> 25.7, cfg3 53.3
// -> 52.5; in the batch kernel it cost 1-3% (not used there)
#ifndef VXM_TB_TAIL_FAST
#define VXM_TB_TAIL_FAST 1
#endif

// K3 batch kernel: the masked tail fast chunk tried where an exact chunk would
// run (r02cj: trace 109.1 -> 110.2 us per 64 cfg2 frames, cfg1 x64 -1.4%: the
// second fast test per tail chunk costs more than the exact chunks it saves)
#ifndef VXM_TB_TAIL_FAST_BATCH
#define VXM_TB_TAIL_FAST_BATCH 0
#endif

// K3 batch kernel: two fast chunks under one chunk-bound test (2 kChunk - 1
// steps ahead) while it holds (r02cm: trace 109.4 -> 111.0 us per 64 cfg2
// frames, cfg1 x64 -1.3%: the rep loop costs what the saved tests do, and the
// looser bound sends more chunks to the single-chunk test)
#ifndef VXM_TB_FAST2
#define VXM_TB_FAST2 0
#endif

// K3 shape by the call's slots: the batch kernel from VXM_TB_BATCH_MIN slots,
// below that the one-warp kernel, each ray as two halves while the call has at
// most VXM_TB_SPLIT_MAX_RAYS rays. r02cg (graph ms per call): batch kernel from
// 16 slots: cfg2 x8 0.0486 -> 0.0509, cfg1 x8 0.0573 -> 0.0615; split up to 64k
// rays: cfg2 x4 0.0430 -> 0.0451; both kept as they are
#ifndef VXM_TB_BATCH_MIN
#define VXM_TB_BATCH_MIN 8
#endif
#ifndef VXM_TB_SPLIT_MAX_RAYS
#define VXM_TB_SPLIT_MAX_RAYS 32768
#endif

// K3: the key REDs carry an L2 evict-last policy (K4 reads the keys next).
// r02de, three alternating reps: graph frames/s cfg2 x64 +0.4%, cfg1 x64
// +0.2%, bench value inconclusive (380.9k / 383.4k / 382.5k against 383.5k /
// 377.4k / 315.9k with an outlier): within noise, kept off
#ifndef VXM_TB_RED_HINT
#define VXM_TB_RED_HINT 0
#endif
#ifndef VXM_TB_MINB
#define VXM_TB_MINB 20
#endif
#ifndef VXM_TB_FAST
#define VXM_TB_FAST true
#endif
// Batch ray-cast dedup per step of a chunk: bit j set = match.any over the
// warp for step j, clear = the lane+1 / lane+8 neighbours by two shuffles.
// Measured (K3 us per 64 frames, masks 0xF / 0x5 / 0x1 / 0x0): cfg2 (11,439
// rays) 127.9 / 120.9 / 120.7 / 122.4, where match.any saturates the MIO
// queue (ncu mio_throttle 15x cfg1's); cfg1 (19,239 rays) 186.4 / 194.6 /
// 195 / 198.7; cfg3 (76k rays) 299 / 305 / 308 / 311. Bundles of at least
// VXM_TB_MATCH_RAYS rays take the large mask.
// Re-swept at the final round-2 state (profiles/r02cu_knobs_ab.txt,
// r02cx_knobs_ab.txt; bench frames/s at 50 steps, two reps, default 380k):
// 16 / 24 K3 blocks per SM 365k / 370k, 4 branches 369k, 8 merge rows per
// warp 364-368k, small-bundle mask 0x1 / 0x4 367-373k / 377-378k, near mask
// 0x5 378-380k, K4 at 5 blocks per SM 379k: the defaults stay.
#ifndef VXM_TB_MATCH_LARGE
#define VXM_TB_MATCH_LARGE 0xF
#endif
#ifndef VXM_TB_MATCH_SMALL
#define VXM_TB_MATCH_SMALL 0x5
#endif
// the same for the near-field chunks (no occupancy loads): match.any on every
// step for small bundles (cfg2 ray cast -0.8%), on the first step only for
// large ones (cfg3 -2%); r02bg / r02bh
#ifndef VXM_TB_NEAR_MATCH_LARGE
#define VXM_TB_NEAR_MATCH_LARGE 0x1
#endif
#ifndef VXM_TB_NEAR_MATCH_SMALL
#define VXM_TB_NEAR_MATCH_SMALL 0xF
#endif
#ifndef VXM_TB_MATCH_RAYS
#define VXM_TB_MATCH_RAYS 16384
#endif

// Also measured for the fast chunks and not kept (same B200, 64 cfg2 streams,
// within noise): each cell's occupancy load and dedup written right after the
// step that makes it (ptxas schedules both forms alike), and the axis choice
// from three independent compares (ptxas re-chains them).

// Also measured and not kept: lanes without a write sending an unpredicated
// generic RED to a per-lane shared-memory word (no branch around the RED;
// ptxas wraps every predicated RED in one): the generic atomics made the
// batch ray cast 17% slower (130 -> 152 us per 64 cfg2 frames).

// Also measured and not kept: capping the batch ray-cast blocks resident per
// SM with dynamic shared memory so that the other branches' kernels fit
// beside them (12 or 16 blocks instead of 20: 323k -> 267k / 286k frames/s,
// the shared-memory carve-out also shrinks L1 for the occupancy loads), and 4
// graph branches again after the round-2 ray cast (-2%).

// Also measured and not kept: finished rays parked on a per-slot sentinel
// occupancy byte (always the frame's epoch) so that a warp keeps taking fast
// chunks after its first lane ends: K3 115.5 -> 123 us per 64 cfg2 frames
// (more chunks run with few live lanes, and the mutable step increments
// spill at 48 registers).

// x-rows per warp of the direct-load K4 grid when the batch fills the GPU
// many times over (a multiple of kRowsPerWarp = 4); the flat no-x-shift path
// takes its 16-cell chunks over the same grid, so fewer warps amortise the
// per-warp set-up and counter reduction (31% of K4's instructions at 4 rows
// per warp) over more chunks. Measured, 64 cfg2 streams (K4 us / bench
// frames/s): 4 rows 51 / 331k, 8 rows 51 / 333k, 16 rows 46 / 349k, 32 rows
// 48 / 335k; a 48-register cap (VXM_MERGE_MINB 5) 44 / 349k.
#ifndef VXM_MERGE_RPW
#define VXM_MERGE_RPW 16
#endif
// resident blocks per SM the direct-load K4 is compiled for (register cap):
// 4 -> 64 registers; without a cap ptxas took 80 and K4 lost its rows-per-warp
// gain (52 us, 324k frames/s); 5 -> 48 registers with a small spill (equal)
// flat K4: the merged local grid stored with the streaming hint (it is read
// again only by the next frame's K4) instead of a plain store. r02da, three
// alternating reps, bench frames/s at 50 steps: 379.7k / 380.2k / 381.0k ->
// 381.1k / 380.8k / 381.6k; cfg1 x64 234.6-235.2k -> 235.5-235.7k (kept)
#ifndef VXM_MERGE_STCS
#define VXM_MERGE_STCS 1
#endif
#ifndef VXM_MERGE_MINB
#define VXM_MERGE_MINB 4
#endif
// resident blocks per SM the TMA-staged K1 is compiled for (register cap):
// 4 -> 64 registers (uncapped: 77, 3 blocks per SM): +2% frames/s; 5 and 6
// (48 / 40 registers) spill and slow K1 itself
// K1: the depth tiles' bulk copies carry an L2 evict-first policy (each
// frame is read once) so they do not displace the occupancy bytes and keys
// the other branches' kernels work on. r02dc, three alternating reps, bench
// frames/s at 50 steps: 381.5k / 381.8k / 381.4k -> 383.4k / 383.5k / 384.5k,
// populate+dilate 55.6 -> 54.7 us per 64 cfg2 frames (kept)
#ifndef VXM_POP_EVICT_FIRST
#define VXM_POP_EVICT_FIRST 1
#endif
#ifndef VXM_POP_MINB
#define VXM_POP_MINB 4
#endif

// Also measured and not kept: K1 ORing raw centre bits into the dilation's bit
// plane (no centre bytes, no pack phase in K2) with K5 clearing the plane for
// the next frame: K2 no faster and the clearing stores in K5 lengthen every
// branch's chain (355k -> 326k frames/s).

// Longest x-row (cells, dx % 4 == 0) merged by the direct-load K4 (flat
// chunks for frames without an x shift, per-row loops otherwise); longer or
// odd rows take the TMA-staged K4. 1024 (round 2): 16 cfg3 streams (200-cell
// rows) merge in 82 instead of 110 us, 35.5k -> 39.0k frames/s; 128 before.
// K1 dense path: pixels of a quad transformed VXM_POP_BATCH at a time
// (interleaved fp64 chains; 0: one after another). r02bt, cfg1 x64 frames/s:
// 0 230.0k, 2 237.8k, 4 239.2k; K1+K2 88.6 -> 78.3 -> 76.3 us
#ifndef VXM_POP_BATCH
#define VXM_POP_BATCH 4
#endif

// K1 dense path: a warp whose batched tile deferred pixels on more than this
// many lanes (points on voxel faces) takes its remaining tiles one pixel at a
// time (r02by: the batch with deferral alone ran the corridor trajectory at
// 174k frames/s vs 209k one pixel at a time; box scenes the other way round)
#ifndef VXM_POP_SERIAL_LANES
#define VXM_POP_SERIAL_LANES 8
#endif

// ... and every warp starts one pixel at a time when more than this percentage
// of the warps of the slot's previous K1 found face-heavy first tiles
#ifndef VXM_POP_HINT_PCT
#define VXM_POP_HINT_PCT 75
#endif

// K1 compacting path: list entries per lane transformed together (0: one at a
// time). r02bu, cfg2 x64 K1+K2 stage: 0 57.1 us, 2 55.8 us, 4 56.8 us
#ifndef VXM_POP_CBATCH
#define VXM_POP_CBATCH 2
#endif

// K4 flat path: chunk coordinates advanced by the grid stride (1) or two
// division pairs per chunk (0). r02cn: merge stage 45.1 -> 43.0 us per 64 cfg2
// frames (quick_time), bench 46.9 -> 45.6 us and +0.6% frames/s
#ifndef VXM_MERGE_INCR
#define VXM_MERGE_INCR 1
#endif

// K4 / chain merges: the four keys of a word decoded with byte permutes (1)
// or one by one (0). r02cq: K4 flat loop 620 -> 572 SASS instructions, bench
// merge stage 45.6 -> 44.7 us per 64 cfg2 frames, frames/s +0.2-0.9%
#ifndef VXM_MERGE4_PRMT
#define VXM_MERGE4_PRMT 1
#endif

// fewest rows per warp of K4 (a lone frame's slot fills the GPU less than once;
// 4 -> a quarter of the blocks: lone cfg1/cfg2/cfg3 frames unchanged, r02br)
#ifndef VXM_MERGE_RPW_MIN
#define VXM_MERGE_RPW_MIN 1
#endif

// Also measured and not kept (r02cs): K2's z-OR as a sliding window over
// kT + 2r registers (one shared load per z instead of 2r + 1, the z loop
// unrolled): fewer instructions, but populate+dilate 55.8 -> 56.8 us.

#ifndef VXM_MERGE_DIRECT_MAX_DX
#define VXM_MERGE_DIRECT_MAX_DX 1024
#endif

// Also measured and not kept: the occupancy bytes of all slots in the
// persisting L2 carve-out (access-policy window on every stream): ray cast
// -2.5%, merge +3%, frames/s unchanged.

// resident blocks per SM the chain-folded multi-frame merge is compiled for
// (5 -> 48 registers instead of 72: one robot at 64 frames per call +1-2%)
#ifndef VXM_SEQ_MINB
#define VXM_SEQ_MINB 5
#endif

// frames of a chain whose loads the multi-frame merge issues together (even;
// 8 at 64 registers: merge 70 -> 79 us, r02bn/r02bp)
// threads per block of the multi-frame merge (VXM_SEQ_MINB counts 256-thread
// blocks' worth of residency; 128: cfg1 64-frame merge 70.6 -> 66.6 us but
// cfg3 89 -> 91 us, calls unchanged within noise, r02bp)
#ifndef VXM_SEQ_THREADS
#define VXM_SEQ_THREADS 256
#endif

#ifndef VXM_SEQ_U
#define VXM_SEQ_U 4
#endif
