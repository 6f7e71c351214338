/* collsight_b200.h — host-side extensions of the drop-in library.
 *
 * Entry points a maintainer of the reference would bind next to collsight.h
 * to feed the B200 engine without going through a JSONL file:
 *   - the packed-record replay of collsight_run_analyze (the same
 *     run_detection + report rendering, records already in host memory);
 *   - the scenario's layout / program / knobs lowered to the engine's plain
 *     C tables (reference ScenarioConfig::build_topology / build_program,
 *     proj/src/scenario.cpp:65-72);
 *   - the JSONL trace codec (reference parse_trace_text / serialize_records,
 *     proj/src/trace.cpp:155-346) producing/consuming packed records.
 */
#ifndef COLLSIGHT_B200_H_
#define COLLSIGHT_B200_H_

#include <stddef.h>
#include <stdint.h>

#include "collsight.h"
#include "csg_engine.h"

#ifdef __cplusplus
extern "C" {
#endif

/* collsight_run_analyze over packed records in host memory (pinned or
 * pageable): H2D, device index, trigger + RCA, reports. */
collsight_status collsight_b200_run_analyze_packed(
    const collsight_scenario* scenario, const csg_packed_record* records,
    size_t n, const char* report_out_path, collsight_result** out);

/* reports_to_jsonl (reference proj/src/runner.cpp:103-169) of engine results
 * from csg_run_detection under the scenario's config: the report bytes a
 * sharded (multi-GPU) caller writes, identical to collsight_run_analyze's.
 * Caller frees with collsight_b200_free. */
collsight_status collsight_b200_results_jsonl(const collsight_scenario* scenario,
                                              const csg_results* results,
                                              char** jsonl_out);

/* Engine tables of a parsed scenario. The returned JSON text describes the
 * layout and program as {"world_size","groups":[{"kind","members"}],
 * "ops":[{"name","group","src","dst","deps"}]}; caller frees with
 * collsight_b200_free. */
collsight_status collsight_b200_scenario_layout_json(
    const collsight_scenario* scenario, char** json_out);
collsight_status collsight_b200_scenario_configs(
    const collsight_scenario* scenario, csg_trigger_config* trigger,
    csg_analysis_config* analysis, uint64_t* seed);

/* build_layout + default_program (proj/src/topology.cpp:80-148,
 * proj/src/program.cpp:25-119) as the JSON above. */
collsight_status collsight_b200_layout_json(int tp, int pp, int dp,
                                            int ranks_per_node,
                                            int channels_per_pair,
                                            int nics_per_node,
                                            uint64_t msg_bytes,
                                            char** json_out);

/* JSONL <-> packed records. Parse errors follow the reference exactly
 * (TraceParseError "line N: ..." -> status 3). */
collsight_status collsight_b200_parse_trace(const char* text, size_t len,
                                            csg_packed_record** out,
                                            size_t* n);
/* packed records -> JSONL in the reference's serialize_records format
 * (proj/src/trace.cpp:189-322), multithreaded; the dropped fields are written
 * as node = rank / ranks_per_node, stuck_ms = 0, total_chunks = gpu_ready, so
 * the text parses back to the same records. Caller frees *text with
 * collsight_b200_free; *len excludes the terminating NUL. */
collsight_status collsight_b200_serialize_trace(const csg_packed_record* records,
                                                size_t n, int32_t ranks_per_node,
                                                char** text, size_t* len);
/* The same text written to a file (a JSONL trace for collsight_run_analyze). */
collsight_status collsight_b200_write_trace(const csg_packed_record* records, size_t n,
                                            int32_t ranks_per_node, const char* path);
void collsight_b200_free(void* p);

/* The engine context the collsight_* calls run on (created on first use on
 * device $COLLSIGHT_B200_DEVICE, default 0), for csg_ctx_stats /
 * csg_ctx_profile / csg_ctx_kernel_stats. */
collsight_status collsight_b200_engine_context(csg_ctx** out);

/* Synthetic trace of the scenario's layout/program/faults in emission order
 * (benchmark input generator, csrc/host/synth.cpp; not the reference
 * simulator). target_records = 0 means no cap; otherwise the earliest
 * target_records records are kept. Caller frees with collsight_b200_free. */
collsight_status collsight_b200_synthesize(const collsight_scenario* scenario,
                                           uint64_t target_records,
                                           csg_packed_record** out, size_t* n);
/* Same trace restricted to ranks in [rank_lo, rank_hi): one shard's records
 * in emission order (rank-range sharding, csg_ctx_comm_init). */
collsight_status collsight_b200_synthesize_ranks(const collsight_scenario* scenario,
                                                 uint64_t target_records,
                                                 int32_t rank_lo, int32_t rank_hi,
                                                 csg_packed_record** out, size_t* n);

/* The same records generated on the store's GPU and appended to the store
 * (*n records): the host schedules the op instances, the device expands
 * every (instance, rank, channel) flow into its records and orders them by
 * emission (synth_gpu.cu). Byte-identical to collsight_b200_synthesize_ranks. */
collsight_status collsight_b200_synthesize_store(const collsight_scenario* scenario,
                                                 uint64_t target_records,
                                                 int32_t rank_lo, int32_t rank_hi,
                                                 csg_store* store, uint64_t* n);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* COLLSIGHT_B200_H_ */
