// dpd_sched.h -- host runtime of the step pipeline: a GPU-aware task
// scheduler and the asynchronous I/O worker of the compute / postprocess split.
//
// PAPER.md §3.4:
//   * "a GPU-aware task scheduler based on the Kahn's topological sorting algorithm, that
//     supports task execution on concurrent CUDA streams" -> TaskGraph: named
//     tasks on stream slots, dependency edges, Kahn order (cycles rejected), cross-stream
//     edges enforced with CUDA events, same-stream edges by stream order;
//   * "One of the tasks, called compute task, performs the actual time-stepping on the GPU,
//     while the other one (postprocess task) is responsible for all the heavy I/O"
//      -> IoQueue: one worker thread per context behind a bounded queue (SPEC
//     depth configurable, default 4; depth 0 = synchronous; a full queue blocks
//     the submitter, nothing is dropped; a worker error surfaces at the next submit or at
//     close, which drains every pending item first).
// B200 mapping: the "postprocess task" is a host thread of the same process (one process per
// GPU), fed by device-to-host copies on a copy stream into pinned slots, so the disk never
// stalls the compute stream.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace dpd {

// ---------------------------------------------------------------------------------------
// TaskGraph
// ---------------------------------------------------------------------------------------
struct TaskGraph {
    using Fn = std::function<int(cudaStream_t)>;
    struct Task {
        std::string name;
        int slot = 0;             // stream slot the task is issued on
        Fn fn;                    // issues the task's work (kernels, copies, collectives)
        std::vector<int> pred, succ;
    };
    std::vector<Task> tasks;
    std::vector<int> order; // Kahn order, valid after build() == 0
    std::vector<cudaEvent_t> done; // per task, recorded when a successor runs on another slot

    ~TaskGraph()
    {
        for (cudaEvent_t e : done)
            if (e) cudaEventDestroy(e);
    }

    int add(const std::string &name, int slot, Fn fn = nullptr)
    {
        Task t;
        t.name = name;
        t.slot = slot;
        t.fn = std::move(fn);
        tasks.push_back(std::move(t));
        order.clear();
        return (int)tasks.size() - 1;
    }

    // `before` must complete before `after` starts.  -1 on bad ids or a self edge.
    int edge(int before, int after)
    {
        const int n = (int)tasks.size();
        if (before < 0 || after < 0 || before >= n || after >= n || before == after) return -1;
        tasks[before].succ.push_back(after);
        tasks[after].pred.push_back(before);
        order.clear();
        return 0;
    }

    // Kahn's algorithm (Kahn 1962): repeatedly emit a task with no unemitted predecessor; among
    // ready tasks the earliest added goes first, so the issue order is deterministic and
    // follows insertion order wherever the edges allow.  -1 if the edges contain a cycle.
    int build()
    {
        const int n = (int)tasks.size();
        std::vector<int> indeg(n, 0);
        for (const Task &t : tasks)
            for (int s : t.succ) ++indeg[s];
        std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
        for (int i = 0; i < n; ++i)
            if (indeg[i] == 0) ready.push(i);
        order.clear();
        while (!ready.empty()) {
            const int u = ready.top();
            ready.pop();
            order.push_back(u);
            for (int s : tasks[u].succ)
                if (--indeg[s] == 0) ready.push(s);
        }
        if ((int)order.size() != n) {
            order.clear();
            return -1;
        }
        return 0;
    }

    // Issue every task in Kahn order on streams[slot]; a predecessor on another slot is
    // awaited with its completion event (cudaStreamWaitEvent: no host blocking).  Returns the
    // first non-zero task result, or -2 on a CUDA error.
    int run(const cudaStream_t *streams)
    {
        if (order.size() != tasks.size() && build() != 0) return -1;
        if (done.size() != tasks.size()) {
            for (cudaEvent_t e : done)
                if (e) cudaEventDestroy(e);
            done.assign(tasks.size(), nullptr);
            for (size_t i = 0; i < tasks.size(); ++i)
                if (cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess) return -2;
        }
        for (int u : order) {
            const Task &t = tasks[u];
            cudaStream_t st = streams[t.slot];
            for (int p : t.pred)
                if (tasks[p].slot != t.slot && cudaStreamWaitEvent(st, done[p], 0) != cudaSuccess) return -2;
            if (t.fn) {
                const int rc = t.fn(st);
                if (rc) return rc;
            }
            bool cross = false;
            for (int s : t.succ) cross = cross || tasks[s].slot != t.slot;
            if (cross && cudaEventRecord(done[u], st) != cudaSuccess) return -2;
        }
        return 0;
    }
};

// ---------------------------------------------------------------------------------------
// IoQueue: bounded queue + one worker thread
// ---------------------------------------------------------------------------------------
class IoQueue {
public:
    using Job = std::function<int(std::string &err)>; // 0 on success, else sets err

    explicit IoQueue(int depth) : depth_(depth)
    {
        if (depth_ > 0) worker_ = std::thread([this] { loop(); });
    }
    ~IoQueue() { close(); }

    // Enqueue (blocks while `depth` jobs are pending); depth 0 runs the job inline.  Returns
    // 0, or -1 with the first error of an earlier job (reported once).
    int submit(Job job, std::string &err)
    {
        if (take_error(err)) return -1;
        if (depth_ == 0) {
            std::string e;
            if (job(e) != 0) {
                err = e;
                return -1;
            }
            std::lock_guard<std::mutex> lk(m_);
            ++done_;
            return 0;
        }
        std::unique_lock<std::mutex> lk(m_);
        cv_space_.wait(lk, [this] { return (int)q_.size() < depth_ || stop_; });
        if (stop_) {
            err = "I/O queue closed";
            return -1;
        }
        q_.push_back(std::move(job));
        cv_work_.notify_one();
        return 0;
    }

    // Jobs queued or running.
    int64_t pending()
    {
        std::lock_guard<std::mutex> lk(m_);
        return (int64_t)q_.size() + (busy_ ? 1 : 0);
    }
    // Jobs that finished successfully.
    int64_t completed()
    {
        std::lock_guard<std::mutex> lk(m_);
        return done_;
    }

    // Drain every pending job, join the worker; 0 or -1 with the first unreported error.
    int close(std::string *err = nullptr)
    {
        if (worker_.joinable()) {
            {
                std::lock_guard<std::mutex> lk(m_);
                stop_ = true;
            }
            cv_work_.notify_all();
            cv_space_.notify_all();
            worker_.join();
        }
        std::string e;
        if (take_error(e)) {
            if (err) *err = e;
            return -1;
        }
        return 0;
    }

    // Block until every submitted job has finished (the queue stays open).
    void drain()
    {
        std::unique_lock<std::mutex> lk(m_);
        cv_idle_.wait(lk, [this] { return q_.empty() && !busy_; });
    }

private:
    void loop()
    {
        for (;;) {
            Job job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_work_.wait(lk, [this] { return !q_.empty() || stop_; });
                if (q_.empty()) return; // stop_ and drained
                job = std::move(q_.front());
                q_.pop_front();
                busy_ = true;
            }
            cv_space_.notify_one();
            std::string e;
            const int rc = job(e);
            {
                std::lock_guard<std::mutex> lk(m_);
                busy_ = false;
                if (rc == 0) ++done_;
                if (rc != 0 && err_.empty()) err_ = e.empty() ? "I/O job failed" : e;
            }
            cv_idle_.notify_all();
        }
    }

    bool take_error(std::string &err)
    {
        std::lock_guard<std::mutex> lk(m_);
        if (err_.empty()) return false;
        err = err_;
        err_.clear();
        return true;
    }

    const int depth_;
    std::deque<Job> q_;
    std::mutex m_;
    std::condition_variable cv_work_, cv_space_, cv_idle_;
    std::thread worker_;
    std::string err_;
    bool stop_ = false, busy_ = false;
    int64_t done_ = 0;
};

} // namespace dpd
