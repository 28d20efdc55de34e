/* The communicator C ABI from plain C (no CUDA headers, no C++): what a Go /
 * Java / Rust host binding of the multi-rank path does.
 *
 * Two processes (fork before any CUDA call), one rank each, on the default
 * device (a multi-GPU launcher gives each process its GPU with
 * CUDA_VISIBLE_DEVICES; on a one-GPU box both share it and the communicator
 * waits on the host instead of in a kernel). Bootstrap = each rank writes its
 * gq_comm_handle blob to a file the other reads (any out-of-band channel
 * works: sockets, MPI, an RPC). Then one gq_comm_mean call per rank and a
 * cross-check: both ranks' decoded means must equal the single-device
 * gq_mean_inproc of the same two shards, bit for bit.
 *
 *   cc -O2 -I include integration/comm_example.c -Lpaper_2305_18627_b200 -lgq_b200 -o comm_example
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/wait.h>
#include <unistd.h>

#include "gq_b200.h"

#define NR 2
#define D (1u << 16)

static int die(const char* what, int rc) {
  fprintf(stderr, "%s failed (%d): %s\n", what, rc, gq_last_error());
  return 1;
}
#define OK(call)                      \
  do {                                \
    int rc_ = (call);                 \
    if (rc_ != GQ_OK) return die(#call, rc_); \
  } while (0)

/* worker w's synthetic gradient: a fixed LCG, centred */
static void shard(uint32_t w, float* x) {
  uint64_t s = 0x9e3779b97f4a7c15ull * (w + 1);
  for (uint32_t j = 0; j < D; ++j) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x[j] = (float)((double)(s >> 40) / (double)(1ull << 24) - 0.5);
  }
}

static gq_config config(void) {
  gq_config c;
  memset(&c, 0, sizeof(c));
  c.workers = NR;
  c.kind = GQ_KIND_EXPONENTIAL;
  c.s = 4;
  c.norm_q = GQ_NORM_INF;
  c.norm_p = GQ_NORM_INF;
  c.width_bits = 4;
  c.topo = GQ_TOPO_TREE;
  c.seed = 42;
  return c;
}

static void path(char* out, size_t n, const char* dir, const char* kind, int r) {
  snprintf(out, n, "%s/%s%d.bin", dir, kind, r);
}

static int wait_read(const char* p, void* buf, size_t bytes) {
  for (int tries = 0; tries < 60000; ++tries) {
    FILE* f = fopen(p, "rb");
    if (f) {
      size_t got = fread(buf, 1, bytes, f);
      fclose(f);
      if (got == bytes) return 0;
    }
    usleep(1000);
  }
  return -1;
}

static int write_file(const char* p, const void* buf, size_t bytes) {
  char tmp[512];
  snprintf(tmp, sizeof(tmp), "%s.tmp", p);
  FILE* f = fopen(tmp, "wb");
  if (!f || fwrite(buf, 1, bytes, f) != bytes) return -1;
  fclose(f);
  return rename(tmp, p);  /* the reader never sees a partial file */
}

static int rank_main(int r, const char* dir) {
  gq_config cfg = config();
  gq_comm* comm = NULL;
  OK(gq_comm_init((uint32_t)r, NR, &cfg, D, &comm));
  const size_t hb = gq_comm_handle_bytes();
  unsigned char* blobs = calloc(NR, hb);
  OK(gq_comm_handle(comm, blobs + r * hb));
  char p[512];
  path(p, sizeof(p), dir, "handle", r);
  if (write_file(p, blobs + r * hb, hb)) return die("write handle", -1);
  for (int q = 0; q < NR; ++q) {
    path(p, sizeof(p), dir, "handle", q);
    if (q != r && wait_read(p, blobs + q * hb, hb)) return die("read peer handle", -1);
  }
  OK(gq_comm_connect(comm, blobs));

  float* host = malloc(D * sizeof(float));
  shard((uint32_t)r, host);
  void *x = NULL, *mean = NULL, *err = NULL;
  OK(gq_malloc(D * sizeof(float), &x));
  OK(gq_malloc(D * sizeof(float), &mean));
  OK(gq_malloc(4, &err));
  OK(gq_memset(err, 0, 4, NULL));
  OK(gq_memcpy(x, host, D * sizeof(float), NULL));
  const void* shards[1] = {x};
  OK(gq_comm_mean(comm, shards, GQ_DTYPE_F32, 7, (float*)mean, NULL, NULL, 0.0f, NULL, (uint32_t*)err, NULL));
  OK(gq_sync(comm, (uint32_t*)err, NULL));
  OK(gq_memcpy(host, mean, D * sizeof(float), NULL));
  OK(gq_stream_sync(NULL));
  path(p, sizeof(p), dir, "mean", r);
  if (write_file(p, host, D * sizeof(float))) return die("write mean", -1);
  /* keep the mapping alive until every rank has its result */
  for (int q = 0; q < NR; ++q) {
    float* tmp = malloc(D * sizeof(float));
    path(p, sizeof(p), dir, "mean", q);
    if (wait_read(p, tmp, D * sizeof(float))) return die("wait peer mean", -1);
    free(tmp);
  }
  gq_comm_destroy(comm);
  return 0;
}

/* the same two shards through the single-device path */
static int reference_mean(float* out) {
  gq_config cfg = config();
  void *x[NR], *lanes[NR], *mean, *stats, *norm, *ws, *err;
  float* host = malloc(D * sizeof(float));
  for (int w = 0; w < NR; ++w) {
    shard((uint32_t)w, host);
    OK(gq_malloc(D * sizeof(float), &x[w]));
    OK(gq_memcpy(x[w], host, D * sizeof(float), NULL));
    OK(gq_malloc(gq_lane_bytes(D, 4) + 256, &lanes[w]));
    OK(gq_memset(lanes[w], 0, gq_lane_bytes(D, 4) + 256, NULL));
  }
  OK(gq_malloc(D * sizeof(float), &mean));
  OK(gq_malloc(8 * NR, &stats));
  OK(gq_malloc(8, &norm));
  OK(gq_malloc(gq_norm_workspace_bytes(NR, D), &ws));
  OK(gq_memset(ws, 0, gq_norm_workspace_bytes(NR, D), NULL));
  OK(gq_malloc(4, &err));
  OK(gq_memset(err, 0, 4, NULL));
  OK(gq_mean_inproc((const void* const*)x, GQ_DTYPE_F32, D, &cfg, 7, lanes, NULL, (float*)mean, NULL, 0.0f,
                    (double*)stats, (double*)norm, ws, (uint32_t*)err, NULL));
  OK(gq_check((uint32_t*)err, NULL));
  OK(gq_memcpy(out, mean, D * sizeof(float), NULL));
  OK(gq_stream_sync(NULL));
  return 0;
}

int main(void) {
  char dir[] = "/tmp/gq_comm_example_XXXXXX";
  if (!mkdtemp(dir)) return die("mkdtemp", -1);
  pid_t pids[NR];
  for (int r = 0; r < NR; ++r) {
    pids[r] = fork();
    if (pids[r] == 0) _exit(rank_main(r, dir));
  }
  int bad = 0;
  for (int r = 0; r < NR; ++r) {
    int st = 0;
    waitpid(pids[r], &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) bad = 1;
  }
  if (bad) {
    printf("FAIL comm_example: a rank failed\n");
    return 1;
  }
  float* want = malloc(D * sizeof(float));
  float* got = malloc(D * sizeof(float));
  if (reference_mean(want)) return 1;
  for (int r = 0; r < NR; ++r) {
    char p[512];
    path(p, sizeof(p), dir, "mean", r);
    if (wait_read(p, got, D * sizeof(float)) || memcmp(got, want, D * sizeof(float)) != 0) {
      printf("FAIL comm_example: rank %d mean differs from gq_mean_inproc\n", r);
      return 1;
    }
  }
  printf("PASS comm_example: 2 processes, gq_comm over CUDA IPC, means bit-identical to gq_mean_inproc (d=%u)\n", D);
  for (int r = 0; r < NR; ++r) {
    char p[512];
    path(p, sizeof(p), dir, "handle", r);
    unlink(p);
    path(p, sizeof(p), dir, "mean", r);
    unlink(p);
  }
  rmdir(dir);
  return 0;
}
