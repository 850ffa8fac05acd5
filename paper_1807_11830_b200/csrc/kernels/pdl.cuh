// pdl.cuh -- programmatic dependent launch (PDL) hooks shared by every kernel.
//
// GraphProcess::capture() turns the kernel -> kernel edges of a process graph
// into programmatic edges (processes.cpp), so a kernel's CTAs are launched
// while its predecessor drains and the launch latency + prologue (twiddle
// registers) overlap the predecessor's tail.  Every kernel therefore
//   1. lets its successor launch once all of its own CTAs are resident
//      (griddepcontrol.launch_dependents at entry), and
//   2. waits for its predecessor's completion and memory flush
//      (griddepcontrol.wait) before it touches any buffer that predecessor may
//      read or write -- only immutable init-time tables (twiddles) are read
//      before the wait.
// Both instructions are no-ops when the kernel was launched normally.
#pragma once

namespace hetreco::dev {

__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace hetreco::dev
