"""L2 flush between timed steps (bench.py and tools/): write a 256 MiB buffer (larger than the 126 MB L2), then read a
clean 256 MiB buffer.  The write alone evicts everything but leaves ~126 MB of the flush buffer's DIRTY lines in L2,
and the next kernel then pays their write-back inside its timed region (bench/micro/hbm_stream.cu: a 268 MB bulk-copy
stream takes 57 us after a write-only flush and 45 us after write + read; profiles/hbm_stream_r2.txt).  After the
read the L2 holds only clean lines of the flush buffer: the timed step starts cold with nothing of its own cached and
nothing else to write back."""
import torch


class L2Flush:
    def __init__(self, device):
        self.dirty = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        self.clean = torch.zeros((256 << 20) // 4, dtype=torch.int32, device=device)
        self.sink = torch.empty((), dtype=torch.int64, device=device)

    def __call__(self):
        self.dirty.zero_()
        torch.sum(self.clean, dim=0, dtype=torch.int64, out=self.sink)

    def zero_(self):  # drop-in for the former `flush.zero_()`
        self()

    describe = ("flushed before every timed step: 256 MiB write, then a 256 MiB read of a clean buffer (no dirty flush "
                "lines left to write back inside the step); per-step CUDA events")
