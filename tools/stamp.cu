// stamp.cu -- one thread writes %globaltimer to out[i] (a stream-ordered
// device timestamp between two launches).  Built to tools/stamp.cubin.
extern "C" __global__ void stamp(unsigned long long* out, int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  out[i] = t;
}
