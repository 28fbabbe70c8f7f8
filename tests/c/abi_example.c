/* Plain C client of the C-ABI, compiled against include/cfpq.h (no Python, no torch).
 *   abi_example layout   print offsetof/sizeof of cfpq_options (checked against the ctypes
 *                        mirror by tests/test_abi.py, CPU)
 *   abi_example run      the paper's worked example through the raw ABI on the
 *                        current CUDA device: 6 loop bodies ("k = 6"), R_S =
 *                        {(0,0), (0,2), (1,2)}, the two-call size query, a NULL
 *                        argument and an out-of-range edge (tests/test_gpu_abi_c.py)   */
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "cfpq.h"

#define FIELD(f) printf("%s %zu\n", #f, offsetof(cfpq_options, f))

static int fail(const char* what, cfpq_status st) {
    printf("FAIL %s: status %d: %s\n", what, (int)st, cfpq_last_error());
    return 1;
}

int main(int argc, char** argv) {
    if (argc > 1 && strcmp(argv[1], "layout") == 0) {
        printf("sizeof %zu\n", sizeof(cfpq_options));
        FIELD(semantics); FIELD(schedule); FIELD(path_policy); FIELD(account_work);
        FIELD(max_iterations); FIELD(cuda_stream); FIELD(world_size); FIELD(rank);
        FIELD(nccl_unique_id); FIELD(log_capacity); FIELD(solo_threshold); FIELD(record_times);
        FIELD(max_ctas); FIELD(reserved_emulate); FIELD(cell_set); FIELD(tensor_format);
        FIELD(dense_launch); FIELD(diag_flags); FIELD(grid_rows); FIELD(grid_cols);
        FIELD(rows_list_capacity); FIELD(exchange);
        return 0;
    }
    /* G': S=0, S1..S6 = 1..6; labels subClassOf_r=0, subClassOf=1, type_r=2, type=3 */
    const int32_t bin[] = {0, 1, 5, 0, 3, 6, 0, 1, 2, 0, 3, 4, 5, 0, 2, 6, 0, 4};
    const int32_t term[] = {1, 0, 2, 1, 3, 2, 4, 3};
    const int32_t edges[] = {0, 0, 0, 0, 2, 1, 1, 2, 2, 2, 1, 0, 2, 3, 2};   /* reading c1 */
    cfpq_grammar* g = NULL;
    cfpq_graph* d = NULL;
    cfpq_result* r = NULL;
    cfpq_status st;
    if ((st = cfpq_grammar_create(7, 4, bin, 6, term, 4, &g)) != CFPQ_OK) return fail("grammar", st);
    if ((st = cfpq_graph_create(3, edges, 5, 0, NULL, &d)) != CFPQ_OK) return fail("graph", st);
    int policies[] = {1, 2, 3};
    for (int q = 0; q < 3; ++q) {
        cfpq_options o;
        cfpq_options_default(&o);
        o.path_policy = policies[q];
        if ((st = cfpq_closure(g, d, &o, &r)) != CFPQ_OK) return fail("closure", st);
        int64_t it = 0, cnt = 0, written = 0;
        cfpq_result_iterations(r, &it);
        if (it != 6) { printf("FAIL iterations %lld\n", (long long)it); return 1; }
        if ((st = cfpq_result_count(r, 0, &cnt)) != CFPQ_OK) return fail("count", st);
        int32_t pairs[6] = {0};
        if (cnt != 3) { printf("FAIL |R_S| = %lld\n", (long long)cnt); return 1; }
        if (cfpq_result_pairs(r, 0, pairs, 2, 0, &written) != CFPQ_E_INVAL) { printf("FAIL capacity check\n"); return 1; }
        if ((st = cfpq_result_pairs(r, 0, pairs, 3, 0, &written)) != CFPQ_OK) return fail("pairs", st);
        const int32_t exp[6] = {0, 0, 0, 2, 1, 2};
        if (written != 3 || memcmp(pairs, exp, sizeof(exp)) != 0) { printf("FAIL R_S\n"); return 1; }
        cfpq_result_destroy(r);
        r = NULL;
    }
    if (cfpq_closure(g, NULL, NULL, &r) != CFPQ_E_INVAL) { printf("FAIL NULL args\n"); return 1; }
    const int32_t bad[] = {0, 0, 7};
    cfpq_graph* db = NULL;
    if ((st = cfpq_graph_create(3, bad, 1, 0, NULL, &db)) != CFPQ_OK) return fail("graph bad", st);
    cfpq_options o;
    cfpq_options_default(&o);
    if (cfpq_closure(g, db, &o, &r) != CFPQ_E_INVAL) { printf("FAIL out-of-range edge accepted\n"); return 1; }
    cfpq_graph_destroy(db);
    cfpq_graph_destroy(d);
    cfpq_grammar_destroy(g);
    printf("OK %s\n", cfpq_version());
    return 0;
}
