/* The reference's C-interface test sequence (/root/reference/proj/tests/
 * test_capi.cpp:35-143: versions and presets, trace lifecycle, simulate and
 * tune, error paths) as a plain C program, compiled unchanged against EITHER
 * the reference's include/warpred.h or this repo's include/warpred_gpu.h
 * (-DWARPRED_GPU_HEADER) and linked against either library. It prints one
 * JSON object with every wr_simulate result of a policy/threshold sweep, so
 * tests/test_capi_shim.py can run the reference build and the B200 build
 * side by side and compare them field by field.
 *
 *   capi_sequence <tmpdir>           exit status = number of failed checks
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>

#ifdef WARPRED_GPU_HEADER
#include "warpred_gpu.h"
#else
#include "warpred.h"
#endif

static int checks = 0, failed = 0;
#define CHECK(c)                                                            \
  do {                                                                      \
    ++checks;                                                               \
    if (!(c)) {                                                             \
      ++failed;                                                             \
      fprintf(stderr, "CHECK failed at line %d: %s (%s)\n", __LINE__, #c,   \
              wr_last_error());                                             \
    }                                                                       \
  } while (0)

static wr_scene_spec small_scene(void) { /* test_capi.cpp:22-32 */
  wr_scene_spec s;
  wr_scene_spec_init(&s);
  s.num_primitives = 128;
  s.params_per_primitive = 2;
  s.image_width = 32;
  s.image_height = 16;
  s.locality = 0.9;
  s.activity_prob = 0.8;
  s.seed = 99;
  return s;
}

static int exists(const char* p) {
  struct stat st;
  return stat(p, &st) == 0;
}

static void version_and_presets(void) { /* test_capi.cpp:37-54 */
  CHECK(strlen(wr_version()) > 0);
  CHECK(wr_preset_count() == 3);
  int found_big = 0;
  for (int i = 0; i < wr_preset_count(); ++i) {
    wr_machine_config cfg;
    CHECK(wr_machine_preset(wr_preset_name(i), &cfg) == WR_OK);
    if (strcmp(wr_preset_name(i), "rtx4090like") == 0) {
      found_big = 1;
      CHECK(cfg.num_sms == 144);
      CHECK(cfg.rop_units == 176);
    }
  }
  CHECK(found_big);
  wr_machine_config cfg;
  CHECK(wr_machine_preset("nope", &cfg) == WR_ERR_INVALID_ARGUMENT);
  CHECK(strstr(wr_last_error(), "nope") != NULL);
}

static void trace_lifecycle(const char* dir) { /* test_capi.cpp:56-88 */
  const wr_scene_spec scene = small_scene();
  wr_trace* trace = NULL;
  CHECK(wr_trace_generate(&scene, &trace) == WR_OK);
  const int64_t records = wr_trace_record_count(trace);
  CHECK(records > 0);
  char csv[1024], bin[1024], hist[1024], f[2048];
  snprintf(csv, sizeof csv, "%s/t.csv", dir);
  snprintf(bin, sizeof bin, "%s/t.bin", dir);
  snprintf(hist, sizeof hist, "%s/hist", dir);
  CHECK(wr_trace_save(trace, csv, 0) == WR_OK);
  CHECK(wr_trace_save(trace, bin, 1) == WR_OK);
  wr_trace* loaded = NULL;
  CHECK(wr_trace_load(bin, 1, &loaded) == WR_OK);
  CHECK(wr_trace_record_count(loaded) == records);
  wr_trace* from_text = NULL; /* beyond test_capi: the text round trip */
  CHECK(wr_trace_load(csv, 0, &from_text) == WR_OK);
  CHECK(wr_trace_record_count(from_text) == records);
  uint64_t distinct[33], active[33];
  CHECK(wr_trace_histogram_distinct(trace, distinct) == WR_OK);
  CHECK(wr_trace_histogram_active(trace, active) == WR_OK);
  uint64_t total = 0;
  for (int i = 0; i < 33; ++i) total += distinct[i];
  CHECK(total > 0);
  CHECK(wr_trace_write_histograms(trace, hist) == WR_OK);
  snprintf(f, sizeof f, "%s/histogram_distinct.csv", hist);
  CHECK(exists(f));
  snprintf(f, sizeof f, "%s/histogram_active.csv", hist);
  CHECK(exists(f));
  wr_trace_free(from_text);
  wr_trace_free(loaded);
  wr_trace_free(trace);
}

static void simulate_and_tune(const char* dir) { /* test_capi.cpp:90-121 */
  const wr_scene_spec scene = small_scene();
  wr_trace* trace = NULL;
  CHECK(wr_trace_generate(&scene, &trace) == WR_OK);
  wr_machine_config machine;
  CHECK(wr_machine_preset("tiny", &machine) == WR_OK);
  wr_run_metrics native, swb;
  CHECK(wr_simulate(trace, &machine, WR_POLICY_NATIVE, 0, &native) == WR_OK);
  CHECK(native.total_cycles > 0);
  CHECK(native.atomic_requests_to_l2 > 0);
  CHECK(wr_simulate(trace, &machine, WR_POLICY_SW_B, 0, &swb) == WR_OK);
  CHECK(swb.atomic_requests_to_l2 < native.atomic_requests_to_l2);
  wr_tune_report report;
  CHECK(wr_tune(trace, &machine, WR_FAMILY_SW_S, 0, &report) == WR_OK);
  CHECK(report.chosen >= 0 && report.chosen <= 32);
  CHECK(report.reprofile_period == 2000);
  for (int t = 0; t <= 32; ++t)
    CHECK(report.cycles_by_threshold[report.chosen] <= report.cycles_by_threshold[t]);
  char path[4096];
  snprintf(path, sizeof path, "%s/tune.csv", dir);
  CHECK(wr_tune_report_save_csv(&report, path) == WR_OK);
  CHECK(exists(path));
  wr_trace_free(trace);
}

static void error_paths(void) { /* test_capi.cpp:123-143 */
  CHECK(wr_trace_generate(NULL, NULL) == WR_ERR_INVALID_ARGUMENT);
  wr_scene_spec bad = small_scene();
  bad.activity_prob = 7.0;
  wr_trace* trace = NULL;
  CHECK(wr_trace_generate(&bad, &trace) == WR_ERR_INVALID_ARGUMENT);
  CHECK(strstr(wr_last_error(), "activity_prob") != NULL);
  wr_trace* missing = NULL;
  CHECK(wr_trace_load("/no/such/file.csv", 0, &missing) != WR_OK);
  const wr_scene_spec scene = small_scene();
  CHECK(wr_trace_generate(&scene, &trace) == WR_OK);
  wr_machine_config machine;
  CHECK(wr_machine_preset("tiny", &machine) == WR_OK);
  wr_run_metrics m;
  CHECK(wr_simulate(trace, &machine, WR_POLICY_SW_S, 99, &m) == WR_ERR_INVALID_ARGUMENT);
  CHECK(wr_simulate(NULL, &machine, WR_POLICY_NATIVE, 0, &m) == WR_ERR_INVALID_ARGUMENT);
  CHECK(strcmp(wr_last_error(), "null argument") == 0);
  CHECK(wr_trace_record_count(NULL) == -1);
  CHECK(wr_preset_name(3) == NULL);
  wr_trace_free(trace);
}

/* wr_simulate over a policy / threshold sweep of two scenes, printed as JSON
 * for the side-by-side comparison. */
static void sweep(void) {
  wr_scene_spec scenes[2];
  scenes[0] = small_scene();
  wr_scene_spec_init(&scenes[1]);
  scenes[1].num_primitives = 2000;
  scenes[1].params_per_primitive = 9;
  scenes[1].image_width = 128;
  scenes[1].image_height = 64;
  scenes[1].mean_fragment_span = 24.0;
  scenes[1].fragments_per_pixel_mean = 3.0;
  scenes[1].locality = 0.8;
  scenes[1].activity_prob = 0.6;
  scenes[1].seed = 2024;
  const struct { wr_policy_kind k; const char* name; int t; } runs[] = {
      {WR_POLICY_NATIVE, "native", 0}, {WR_POLICY_SW_S, "sw_s", 0}, {WR_POLICY_SW_S, "sw_s", 8},
      {WR_POLICY_SW_S, "sw_s", 16},    {WR_POLICY_SW_S, "sw_s", 32}, {WR_POLICY_SW_B, "sw_b", 0},
      {WR_POLICY_SW_B, "sw_b", 8},     {WR_POLICY_SW_B, "sw_b", 16}, {WR_POLICY_SW_B, "sw_b", 33},
      {WR_POLICY_CCCL, "cccl", 0}};
  wr_machine_config machine;
  CHECK(wr_machine_preset("rtx4090like", &machine) == WR_OK);
  printf("{\"checks\": %d, \"runs\": {", checks);
  for (int s = 0; s < 2; ++s) {
    wr_trace* tr = NULL;
    CHECK(wr_trace_generate(&scenes[s], &tr) == WR_OK);
    for (size_t i = 0; i < sizeof runs / sizeof runs[0]; ++i) {
      wr_run_metrics m;
      memset(&m, 0, sizeof m);
      CHECK(wr_simulate(tr, &machine, runs[i].k, runs[i].t, &m) == WR_OK);
      CHECK(m.total_cycles > 0);
      printf("%s\"s%d:%s:%d\": {\"requests\": %llu, \"instructions\": %llu, \"fp_adds\": %llu, "
             "\"cycles\": %llu}",
             (s || i) ? ", " : "", s, runs[i].name, runs[i].t,
             (unsigned long long)m.atomic_requests_to_l2, (unsigned long long)m.core_instructions,
             (unsigned long long)m.core_fp_adds, (unsigned long long)m.total_cycles);
    }
    wr_trace_free(tr);
  }
}

int main(int argc, char** argv) {
  const char* dir = argc > 1 ? argv[1] : "/tmp";
  if (strlen(dir) > 900) return 99;
  version_and_presets();
  trace_lifecycle(dir);
  simulate_and_tune(dir);
  error_paths();
  sweep();
  printf("}, \"total_checks\": %d, \"failed\": %d}\n", checks, failed);
  return failed;
}
