/*
 * oracle.h — CPU restatement of the reference's layer math (TEST INFRASTRUCTURE).
 *
 * This is the parity checker for the Superpipeline executor, NOT product code:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. Every function restates one reference function
 * (file:line cited against /root/reference/proj/core) in plain C, keeping the
 * reference's exact fp32 evaluation order (separately rounded mul and add, no
 * FMA contraction: build with -ffp-contract=off) so results are bit-identical.
 *
 * Parity pinned: checked against the reference compiled from its own sources
 * (oracle/_ref/libpipesim_ref.so, recipe in oracle/Makefile) and against the
 * golden digests of SURVEY.md Appendix A (tests/golden/golden.json).
 */
#ifndef SP_ORACLE_H
#define SP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* splitmix64 step — model.hpp:40-52 (SplitMix64::next / next_unit). */
uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_unit(uint64_t* state);

/* build_model — model.cpp:23-52. W: n*d*d ([layer][in][out] row-major), b: n*d. */
int orc_build_model(uint64_t seed, int n_layers, int d, float* W, float* b);

/* make_input — model.cpp:186-191. out: rows*d. */
void orc_make_input(uint64_t seed, uint64_t tag, int64_t rows, int d, float* out);

/* layer_forward — model.cpp:54-70. relu: 1 = ReLU, 0 = Identity. */
void orc_layer_forward(int d, const float* W, const float* b, int relu, const float* x,
                       int64_t rows, float* y);

/* layer_backward — model.cpp:72-123. dW/db may be NULL (frozen layers). */
void orc_layer_backward(int d, const float* W, const float* b, int relu, const float* x,
                        const float* dy, int64_t rows, float* dx, float* dW, float* db);

/* mse_loss / mse_grad — model.cpp:131-148. */
float orc_mse_loss(const float* y, const float* t, int64_t count);
void orc_mse_grad(const float* y, const float* t, int64_t count, float* g);

/* apply_sgd — model.cpp:150-155 (caller skips frozen blocks). */
void orc_apply_sgd(float* w, const float* g, int64_t count, float lr);

/* AdamW step (no reference counterpart: the reference trains with apply_sgd). Restates
 * PyTorch's single-tensor AdamW (torch/optim/adamw.py, decoupled weight decay) with every
 * operation separately rounded, in this order:
 *   w *= decay;  m += omb1 * (g - m);  v = v * b2 + (omb2 * g) * g;
 *   w += neg_step * (m / (sqrt(v) / bc2_sqrt + eps))
 * with decay = 1 - lr*wd, omb1 = 1 - b1, omb2 = 1 - b2, neg_step = -lr / (1 - b1^t),
 * bc2_sqrt = sqrt(1 - b2^t), each computed in double and rounded to float once (as PyTorch
 * does with its Python-float scalars). Pinned against torch.optim.AdamW in tests/. */
void orc_adamw(int64_t count, float* w, float* m, float* v, const float* g, float decay,
               float omb1, float b2, float omb2, float bc2_sqrt, float eps, float neg_step);

/* reference_forward — model.cpp:125-129. relu: per-layer flags (NULL = all ReLU). */
void orc_forward(int n_layers, int d, const float* W, const float* b, const int* relu,
                 const float* x, int64_t rows, float* y);

/* reference_train_step — model.cpp:157-184. Mutates W, b in place. frozen/relu may be
 * NULL. Optional outputs (NULL to skip): dW_all n*d*d and db_all n*d (zeros for frozen
 * layers), dx0 rows*d (the input gradient of layer 0). Returns the loss. */
float orc_train_step(int n_layers, int d, float* W, float* b, const int* relu,
                     const int* frozen, const float* x, const float* target, int64_t rows,
                     float lr, float* dW_all, float* db_all, float* dx0);

/* fnv1a64 + digests — engine.cpp:14-31 (fnv1a64, to_hex), :565-581. */
uint64_t orc_fnv1a64(const void* data, uint64_t size, uint64_t h);
/* digest_tensors over n_items tensors of shape [rows, d] stored contiguously. */
uint64_t orc_digest_tensors(int n_items, int64_t rows, int d, const float* values);
/* digest_train(loss, model). */
uint64_t orc_digest_train(float loss, int n_layers, int d, const float* W, const float* b);
void orc_to_hex(uint64_t v, char out[17]);

#ifdef __cplusplus
}
#endif
#endif
