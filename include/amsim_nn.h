/*
 * amsim_nn.h -- C ABI of the NON-approximated layers of a full ApproxTrain
 * training / inference step, in libamsim.so.
 *
 * The paper approximates only the multiplications of Conv2D and Dense
 * ("layers ... that contain multiplications"); batch
 * normalisation, ReLU, pooling, the residual add, the softmax cross-entropy
 * loss and the SGD update run in native FP32 arithmetic.  These kernels are
 * that native part, so a whole training step (PAPER.md:888-942 time whole
 * training steps) runs on the GPU around the AMSim passes of amsim.h.
 *
 * Conventions: as amsim.h -- every tensor is an FP32 (uint8 / int32 where
 * stated) DEVICE pointer owned by the caller, activations NHWC with the
 * channel dimension innermost ("rows" P = N*H*W, channels C); calls
 * validate arguments synchronously (AMSIM_ERR_INVALID_ARG before any launch),
 * enqueue on `stream` and return without synchronising; launch failures
 * return AMSIM_ERR_CUDA.  Results are deterministic (fixed reduction orders,
 * no atomics).  `ws` is caller-owned device scratch of at least
 * amsim_nn_workspace_bytes(P, C) bytes.
 */
#ifndef AMSIM_NN_H
#define AMSIM_NN_H

#include "amsim.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Scratch bytes the per-channel reductions below need for P rows x C channels. */
size_t amsim_nn_workspace_bytes(int64_t P, int32_t C);

/* Batch normalisation, training mode (Ioffe & Szegedy; the BN of the paper's
 * ResNets), fused with an optional residual add and ReLU:
 *   mean_c, var_c over the P rows (biased variance), invstd_c = 1/sqrt(var_c + eps),
 *   y = [relu]( (x - mean_c) * invstd_c * gamma_c + beta_c [+ res] ).
 * save_mean / save_invstd [C] receive the batch statistics for the backward;
 * running_mean / running_var [C] (may be NULL) are updated with `momentum`
 * (r = (1-momentum) r + momentum * stat, unbiased variance).  res may be NULL. */
amsim_status amsim_bn_fwd_train(const float *x, int64_t P, int32_t C, const float *gamma, const float *beta,
                                float eps, const float *res, int relu, float *y, float *save_mean,
                                float *save_invstd, float *running_mean, float *running_var, float momentum,
                                void *ws, size_t ws_bytes, amsim_stream_t stream);

/* Batch normalisation, inference mode: the running statistics replace the
 * batch statistics; same fusion as above. */
amsim_status amsim_bn_fwd_infer(const float *x, int64_t P, int32_t C, const float *gamma, const float *beta,
                                const float *running_mean, const float *running_var, float eps,
                                const float *res, int relu, float *y, amsim_stream_t stream);

/* Backward of amsim_bn_fwd_train.  dz = dy * [y > 0 if relu]; with
 * xhat = (x - mean) * invstd:  dbeta = sum dz, dgamma = sum dz * xhat,
 * dx = gamma * invstd * (dz - dbeta / P - xhat * dgamma / P);
 * dres (may be NULL) receives dz, the gradient of the residual input.
 * y is the forward output (read only when relu). */
amsim_status amsim_bn_bwd(const float *dy, const float *y, const float *x, int64_t P, int32_t C,
                          const float *gamma, const float *save_mean, const float *save_invstd, int relu,
                          float *dx, float *dres, float *dgamma, float *dbeta, void *ws, size_t ws_bytes,
                          amsim_stream_t stream);

/* Bias add + optional ReLU (LeNet-5 conv / dense layers, C13: the bias is
 * added in FP32 outside the approximate product):  y = [relu](x + bias_c).
 * Backward: dx = dy * [y > 0 if relu]; dbias_c = sum over rows of dx.
 * In-place (y == x, dx == dy) is allowed. */
amsim_status amsim_bias_act_fwd(const float *x, int64_t P, int32_t C, const float *bias, int relu, float *y,
                                amsim_stream_t stream);
amsim_status amsim_bias_act_bwd(const float *dy, const float *y, int64_t P, int32_t C, int relu, float *dx,
                                float *dbias, void *ws, size_t ws_bytes, amsim_stream_t stream);

/* Max pooling, window R x S, stride, zero-size padding (padded taps never
 * win), NHWC [N][H][W][C] -> [N][OH][OW][C], OH = (H + 2 pad - R) / stride + 1.
 * argmax [N][OH][OW][C] (uint8) records the winning tap kh * S + kw (first
 * maximum in tap order).  Backward gathers: dx[h][w] = sum of dy over the
 * windows whose argmax is (h, w), in fixed window order.  R * S <= 255. */
amsim_status amsim_maxpool_fwd(const float *x, int32_t N, int32_t H, int32_t W, int32_t C, int32_t R, int32_t S,
                               int32_t stride, int32_t pad, float *y, uint8_t *argmax, amsim_stream_t stream);
amsim_status amsim_maxpool_bwd(const float *dy, const uint8_t *argmax, int32_t N, int32_t H, int32_t W, int32_t C,
                               int32_t R, int32_t S, int32_t stride, int32_t pad, float *dx,
                               amsim_stream_t stream);

/* Global average pooling [N][HW][C] -> [N][C] and its backward
 * dx[n][i][c] = dy[n][c] / HW. */
amsim_status amsim_avgpool_fwd(const float *x, int32_t N, int32_t HW, int32_t C, float *y, amsim_stream_t stream);
amsim_status amsim_avgpool_bwd(const float *dy, int32_t N, int32_t HW, int32_t C, float *dx, amsim_stream_t stream);

/* Softmax cross-entropy over K classes, mean over the N rows, fused with its
 * gradient: loss[0] = mean_n (logsumexp(z_n) - z_n[label_n]),
 * dz = (softmax(z) - onehot(label)) / D with D = grad_denominator, or N when
 * it is 0.  Data-parallel training passes the GLOBAL batch as D, so the
 * all-reduce SUM of the ranks' gradients is the gradient of the global-batch
 * mean loss even with uneven shards.  labels int32 in [0, K); the labels
 * live on the device, so a row with an out-of-range label is not reported: it
 * contributes zero loss and the plain softmax / D gradient.
 * ws >= amsim_nn_workspace_bytes(N, 1).  AMSIM_ERR_INVALID_ARG if D < 0. */
amsim_status amsim_softmax_xent(const float *logits, const int32_t *labels, int32_t N, int32_t K,
                                int32_t grad_denominator, float *loss, float *dlogits, void *ws, size_t ws_bytes,
                                amsim_stream_t stream);

/* out = a + b over n elements (the residual-path gradient sum). */
amsim_status amsim_add(const float *a, const float *b, float *out, int64_t n, amsim_stream_t stream);

/* SGD with momentum and L2 weight decay over a flat parameter buffer:
 *   v = momentum * v + (g + weight_decay * w);  w = w - lr * v. */
amsim_status amsim_sgd_momentum(float *w, const float *g, float *v, int64_t n, float lr, float momentum,
                                float weight_decay, amsim_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* AMSIM_NN_H */
