#include <cstdlib>
// Native step driver of the pipelined trainer.
//
// Replaces the per-batch host loop of orchestrator.Trainer.train_batches (the
// reference's training loop, orchestrator.py:520-560, one Python iteration per
// batch): each step is a pack of the batch's inputs into its pinned staging slot
// (parameter block, counts, int64 seed ids -> int32) followed by a handful of
// CUDA runtime calls — H2D of the staging slot, the sample-half graph on the
// sampling stream, the train-half graph on the training stream (which records
// batch k's loss at d_loss_arr[k]) and, once at the end, one D2H of all the
// losses.  Packing step k right before its launches (not all steps up front)
// lets the device start after the first batch's ~1 us pack instead of after
// the whole call's, so the host never becomes the bottleneck of a step that
// takes ~0.19 ms on the device.
//
// Ordering: the staging buffer of set k % n_sets is refilled (H2D) once batch
// k - n_sets was SAMPLED (the train half reads a private copy the sample half
// makes); the set's blocks are resampled once batch k - n_sets trained; batch k
// trains after its sample half; all streams start after the caller's stream and
// the caller's stream waits for them at the end.
#include <cstring>
#include <vector>

#include "hg_common.cuh"
#include "hg_gnn_internal.h"

extern "C" int hg_pipeline_run(int32_t n_steps, int32_t n_sets, const int64_t* sample_execs,
                               const int64_t* train_execs, void* caller_stream, void* sample_stream,
                               void* train_stream, const int64_t* dev_stage, uint8_t* host_stage,
                               int64_t slot_bytes, int32_t counts_offset, int32_t seeds_offset,
                               const int64_t* bp_rows, const int64_t* host_seed_ptrs, const int32_t* n_seeds,
                               const int32_t* n_div, const float* d_loss_arr, float* host_loss) {
    if (n_steps < 0 || n_sets < 1) { hg_set_error("pipeline_run: bad n_steps / n_sets"); return HG_EINVAL; }
    if (n_steps == 0) return HG_OK;
    if (counts_offset < 8 * HG_BP_WORDS || seeds_offset < counts_offset + 8) {
        hg_set_error("pipeline_run: staging layout overlaps the parameter block");
        return HG_EINVAL;
    }
    for (int k = 0; k < n_steps; ++k) {
        if (n_seeds[k] < 0 || seeds_offset + 4LL * n_seeds[k] > slot_bytes) {
            hg_set_error("pipeline_run: batch %d has %d seeds, more than a staging slot holds", k, n_seeds[k]);
            return HG_EINVAL;
        }
    }
    cudaStream_t cs = (cudaStream_t)caller_stream, ss = (cudaStream_t)sample_stream, st = (cudaStream_t)train_stream;
    std::vector<cudaEvent_t> sampled(n_sets), trained(n_sets), copied(n_sets);
    std::vector<char> has_trained(n_sets, 0), has_sampled(n_sets, 0);
    cudaEvent_t start, end_s, end_t;
    const unsigned fl = cudaEventDisableTiming;
    cudaEventCreateWithFlags(&start, fl);
    cudaEventCreateWithFlags(&end_s, fl);
    cudaEventCreateWithFlags(&end_t, fl);
    for (int k = 0; k < n_sets; ++k) {
        cudaEventCreateWithFlags(&sampled[k], fl);
        cudaEventCreateWithFlags(&trained[k], fl);
        cudaEventCreateWithFlags(&copied[k], fl);
    }
    // staging H2D on its own stream: batch k's copy waits only for the set's
    // staging buffer to be free (batch k - n_sets sampled), so it lands while
    // earlier batches are still being sampled instead of in front of batch k's
    // sample half
    // experiment knob HG_PIPE_H2D_LATE=1: the H2D on the sampling stream after the
    // set's previous train half (the pre-round-2 schedule)
    static const int late_h2d = getenv("HG_PIPE_H2D_LATE") ? atoi(getenv("HG_PIPE_H2D_LATE")) : 0;
    cudaStream_t cp;
    cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking);
    cudaEventRecord(start, cs);
    cudaStreamWaitEvent(ss, start, 0);
    cudaStreamWaitEvent(st, start, 0);
    cudaStreamWaitEvent(cp, start, 0);
    cudaError_t err = cudaSuccess;
    auto pack = [&](int k) {  // the staging slot of batch k: bp | counts | seeds (engine.stage_views)
        uint8_t* slot = host_stage + (int64_t)k * slot_bytes;
        memcpy(slot, bp_rows + (int64_t)k * HG_BP_WORDS, 8 * HG_BP_WORDS);
        const int32_t cnt[2] = {n_seeds[k], n_div[k]};
        memcpy(slot + counts_offset, cnt, sizeof(cnt));
        const int64_t* src = reinterpret_cast<const int64_t*>(host_seed_ptrs[k]);
        int32_t* dst = reinterpret_cast<int32_t*>(slot + seeds_offset);
        for (int i = 0; i < n_seeds[k]; ++i) dst[i] = (int32_t)src[i];
    };
    auto sample = [&](int k) {
        const int set = k % n_sets;
        pack(k);
        // the set's staging buffer is free once its previous SAMPLE half ran (the
        // train half reads the private copy that sample half made), so the H2D of
        // batch k lands while earlier batches are still being sampled; the blocks
        // of the set are free once its previous train half ran
        if (has_sampled[set]) cudaStreamWaitEvent(cp, sampled[set], 0);
        if (has_trained[set]) cudaStreamWaitEvent(ss, trained[set], 0);
        cudaStream_t hs = late_h2d ? ss : cp;
        cudaMemcpyAsync(reinterpret_cast<void*>(dev_stage[set]), host_stage + (int64_t)k * slot_bytes,
                        (size_t)seeds_offset + 4 * (size_t)n_seeds[k], cudaMemcpyHostToDevice, hs);
        if (!late_h2d) {
            cudaEventRecord(copied[set], cp);
            cudaStreamWaitEvent(ss, copied[set], 0);
        }
        const cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(sample_execs[set]), ss);
        if (e != cudaSuccess && err == cudaSuccess) err = e;
        cudaEventRecord(sampled[set], ss);
        has_sampled[set] = 1;
    };
    auto train = [&](int k) {
        const int set = k % n_sets;
        cudaStreamWaitEvent(st, sampled[set], 0);
        const cudaError_t e = cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(train_execs[set]), st);
        if (e != cudaSuccess && err == cudaSuccess) err = e;
        cudaEventRecord(trained[set], st);
        has_trained[set] = 1;
    };
    sample(0);
    for (int i = 0; i < n_steps; ++i) {
        if (i + 1 < n_steps) sample(i + 1);
        train(i);
    }
    // the per-step losses, recorded on the device by each train half: one D2H
    cudaMemcpyAsync(host_loss, d_loss_arr, sizeof(float) * (size_t)n_steps, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(end_s, ss);
    cudaEventRecord(end_t, st);
    cudaStreamWaitEvent(cs, end_s, 0);
    cudaStreamWaitEvent(cs, end_t, 0);
    // destruction of a pending event is deferred by the runtime until it completes
    cudaEventDestroy(start);
    cudaEventDestroy(end_s);
    cudaEventDestroy(end_t);
    for (int k = 0; k < n_sets; ++k) {
        cudaEventDestroy(sampled[k]);
        cudaEventDestroy(trained[k]);
        cudaEventDestroy(copied[k]);
    }
    cudaStreamDestroy(cp);  // deferred until its work completes
    if (err != cudaSuccess) {
        hg_set_error("pipeline_run: graph launch failed: %s", cudaGetErrorString(err));
        return HG_ECUDA;
    }
    return hg_check_launch("pipeline_run");
}
