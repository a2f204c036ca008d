/* orl_demo.c -- one PPO iteration (S1..S10) through the C ABI alone: no Python, no
 * PyTorch.  Plain C99 + the CUDA runtime for device memory.
 *
 *   orl_demo <dir> B T V
 *
 * reads raw little-endian inputs from <dir> (written by tests/test_c_demo.py):
 *   logits_old.bin logits_ref.bin logits_new.bin   bf16 [B,T,V]
 *   tokens.bin int32 [B,T]   lengths.bin int32 [B]   seq_reward.bin f32 [B]
 *   values_old.bin values_new.bin f32 [B,T]
 * runs GAE (gamma 1, lambda 0.95), k1 reward shaping (beta 0.01), global whitening,
 * PPO clip 0.2, value clip 0.2, c1 0.5, in micro-batches of 2 sequences, and prints
 * the status and statistics of orl_finalize as one JSON line, then the per-token
 * logp_new and adv arrays to <dir>/c_logp_new.bin and <dir>/c_adv.bin. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "orl.h"

static void *load(const char *dir, const char *name, size_t bytes) {
    char path[4096];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    FILE *f = fopen(path, "rb");
    if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
    void *h = malloc(bytes);
    if (fread(h, 1, bytes, f) != bytes) { fprintf(stderr, "short read %s\n", path); exit(2); }
    fclose(f);
    void *d = NULL;
    if (cudaMalloc(&d, bytes) != cudaSuccess || cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
        fprintf(stderr, "cuda alloc/copy failed for %s\n", name);
        exit(3);
    }
    free(h);
    return d;
}

static void save(const char *dir, const char *name, const void *d, size_t bytes) {
    char path[4096];
    snprintf(path, sizeof path, "%s/%s", dir, name);
    void *h = malloc(bytes);
    cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost);
    FILE *f = fopen(path, "wb");
    fwrite(h, 1, bytes, f);
    fclose(f);
    free(h);
}

static float *zeros(size_t n) {
    float *d = NULL;
    if (cudaMalloc((void **)&d, n * sizeof(float)) != cudaSuccess) exit(3);
    cudaMemset(d, 0, n * sizeof(float));
    return d;
}

#define CHECK(call)                                                                       \
    do {                                                                                  \
        orl_status s_ = (call);                                                           \
        if (s_ != ORL_OK) {                                                               \
            fprintf(stderr, "%s -> %d: %s\n", #call, (int)s_, orl_last_error(ctx));      \
            return 4;                                                                     \
        }                                                                                 \
    } while (0)

int main(int argc, char **argv) {
    if (argc < 5) { fprintf(stderr, "usage: orl_demo <dir> B T V\n"); return 1; }
    const char *dir = argv[1];
    const int64_t B = atoll(argv[2]), T = atoll(argv[3]), V = atoll(argv[4]);
    const size_t nlog = (size_t)(B * T * V) * 2, ntok = (size_t)(B * T);
    const void *lg[3] = {load(dir, "logits_old.bin", nlog), load(dir, "logits_ref.bin", nlog),
                         load(dir, "logits_new.bin", nlog)};
    const int32_t *tokens = load(dir, "tokens.bin", ntok * 4);
    const int32_t *lengths = load(dir, "lengths.bin", (size_t)B * 4);
    const float *reward = load(dir, "seq_reward.bin", (size_t)B * 4);
    const float *v_old = load(dir, "values_old.bin", ntok * 4);
    const float *v_new = load(dir, "values_new.bin", ntok * 4);
    float *logp_old = zeros(ntok), *logp_ref = zeros(ntok), *kl = zeros(ntok), *shaped = zeros(ntok);
    float *adv = zeros(ntok), *adv_lo = zeros(ntok), *ret = zeros(ntok), *logp_new = zeros(ntok);
    float *ent = zeros(ntok);

    orl_ctx *ctx = NULL;
    if (orl_create(0, 1, 0, NULL, &ctx) != ORL_OK) {
        fprintf(stderr, "orl_create: %s\n", orl_last_error(NULL));
        return 4;
    }
    const int64_t mb = 2;
    CHECK(orl_begin_iteration(ctx, NULL));
    for (int role = 0; role < 2; ++role) {
        for (int64_t s = 0; s < B; s += mb) {          /* S1 old; S1 + S2 + S3 ref */
            orl_rows rows = {B - s < mb ? B - s : mb, T, s, tokens, lengths, NULL};
            orl_logits x = {(const char *)lg[role] + (size_t)(s * T * V) * 2, ORL_BF16, 0, V, T * V, V};
            if (role == 0)
                CHECK(orl_logprobs(ctx, &rows, &x, 1.0f, logp_old, NULL, NULL, NULL, NULL, ORL_KL_K1, 0.0, NULL,
                                   NULL, NULL, NULL));
            else
                CHECK(orl_logprobs(ctx, &rows, &x, 1.0f, logp_ref, NULL, NULL, NULL, logp_old, ORL_KL_K1, 0.01,
                                   reward, kl, shaped, NULL));
        }
    }
    CHECK(orl_advantages(ctx, B, T, lengths, ORL_ADV_GAE, 1.0, 0.95, 1, shaped, v_old, reward, adv, adv_lo, ret,
                         NULL, NULL));                  /* S4 */
    CHECK(orl_whiten_stats(ctx, 1, NULL));              /* S6 + C1 */
    orl_ppo_cfg cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.eps_low = cfg.eps_high = 0.2;
    cfg.eps_value = 0.2;
    cfg.c1 = 0.5;
    cfg.kl_loss_est = ORL_KL_K1;
    cfg.ratio_guard = 30.0;
    for (int64_t s = 0; s < B; s += mb) {               /* S1 + S7..S9 actor */
        orl_rows rows = {B - s < mb ? B - s : mb, T, s, tokens, lengths, NULL};
        orl_logits x = {(const char *)lg[2] + (size_t)(s * T * V) * 2, ORL_BF16, 0, V, T * V, V};
        CHECK(orl_ppo_loss(ctx, &rows, &x, 1.0f, &cfg, logp_old, logp_ref, adv, adv_lo, ret, v_new, v_old, logp_new,
                           ent, NULL, NULL, NULL, NULL, NULL));
    }
    orl_stats st;
    const orl_status fin = orl_finalize(ctx, &cfg, &st, NULL, NULL);  /* S10 + C2 */
    printf("{\"status\": %d, \"n_tokens\": %.17g, \"policy_loss\": %.17g, \"value_loss\": %.17g, "
           "\"entropy\": %.17g, \"kl\": %.17g, \"approx_kl_old\": %.17g, \"clip_frac\": %.17g, "
           "\"value_clip_frac\": %.17g, \"ratio_mean\": %.17g, \"total_loss\": %.17g, \"adv_mean\": %.17g, "
           "\"adv_std\": %.17g, \"launches\": %llu}\n",
           (int)fin, st.n_tokens, st.policy_loss, st.value_loss, st.entropy, st.kl, st.approx_kl_old, st.clip_frac,
           st.value_clip_frac, st.ratio_mean, st.total_loss, st.adv_mean, st.adv_std,
           (unsigned long long)orl_launch_count(ctx));
    save(dir, "c_logp_new.bin", logp_new, ntok * 4);
    save(dir, "c_adv.bin", adv, ntok * 4);
    orl_destroy(ctx);
    return fin == ORL_OK ? 0 : 5;
}
