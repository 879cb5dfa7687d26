/*
 * nif_b200_debug.h -- diagnostic knobs of libnif_b200.so (NOT part of the
 * drop-in ABI in nif_b200.h): kernel-variant selectors and phase-stamp
 * buffers used by tools/ probes and the variant-equivalence tests. The
 * production path never calls them; defaults are the shipped kernels.
 */
#ifndef NIF_B200_DEBUG_H
#define NIF_B200_DEBUG_H

#ifdef __cplusplus
extern "C" {
#endif

/* Diagnostics: when buf != NULL the tcgen05 query kernel records clock64()
 * phase stamps of its first 4 tiles per CTA into buf[cta][4][16].      */
int nif_debug_set_prof(void* buf);
/* Same for the gather (one-tile-per-CTA variant): buf[tile][8].        */
int nif_debug_set_prof_gather(void* buf);
/* Gather hot-path variant: 0 unordered warp-chunk compaction (default;
 * queue order is arbitrary, per-ray results identical), 1 one tile per CTA
 * with look-back (reference order), 2 persistent TMA-pipelined look-back
 * (reference order). All produce the same records.                     */
int nif_debug_set_gather_variant(int v);
/* CTAs per SM of the hot-path gather / fused query grids (0: default) */
int nif_debug_set_gather_grid(int ctas_per_sm);
/* Hot-path gather: this many of each warp's static chunk rounds are handed
 * out on demand instead (one atomic per chunk).                        */
int nif_debug_set_gather_dynamic(int rounds);
/* Diagnostic timelines (%globaltimer, ns) of the hot-path kernels, NULL to
 * disable: gather buf[warp][4] = entry, after the prologue, exit, chunks;
 * fused tcgen05 query buf[cta * G + warpgroup][5] = entry, after the grid
 * dependency wait, after the first tile, exit, tiles.                   */
int nif_debug_set_timeline_gather(void* buf);

int nif_debug_set_timeline_query(void* buf);
int nif_debug_set_query_grid(int ctas_per_sm);
/* Culling statistics of the hot-path gather since the last call (rays,
 * bundle survivors, prefilter survivors, classified hits); only in a
 * library built with -DNIF_GATHER_STATS (tools/gather_stats.py).       */
int nif_debug_gather_stats(unsigned long long* out4);
/* Query-kernel variant (benchmarks / equivalence tests): 0 fused with the
 * A operand in TMEM (default); 1 / 9 shared-memory-operand specialisations
 * (6 / 4 tiles per SM); 2 runtime-shape generic kernel; 11 TMEM operand,
 * one tile per CTA.                                                     */
int nif_debug_set_query_variant(int v);
/* Training fwd/bwd kernel: 0 tiled CTA-GEMM kernel where it applies
 * (shared MLP, width a multiple of 16; 16 rows x 256 threads; default),
 * 1 one row per thread, 2 tiled 32 x 128, 3 tiled 32 x 256.            */
int nif_debug_set_train_variant(int v);

#ifdef __cplusplus
}
#endif
#endif /* NIF_B200_DEBUG_H */
