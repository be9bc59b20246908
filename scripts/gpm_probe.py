"""Does NVML GPM (DRAM_BW_UTIL) work here, and what does 100% mean?"""
import time
import pynvml as N
import torch

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
print("gpm support", N.nvmlGpmQueryDeviceSupport(h).isSupportedDevice)
bw = N.nvmlDeviceGetMemoryBusWidth(h)
mclk = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_MEM)
print("bus width", bw, "max mem clock", mclk, "theoretical GB/s", bw * mclk * 2 / 8 / 1e3)
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
for reps in (10, 40):
    s1, s2 = N.nvmlGpmSampleAlloc(), N.nvmlGpmSampleAlloc()
    torch.cuda.synchronize()
    N.nvmlGpmSampleGet(h, s1)
    t0 = time.perf_counter()
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    N.nvmlGpmSampleGet(h, s2)
    mg = N.c_nvmlGpmMetricsGet_t()
    mg.version = N.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = 2
    mg.sample1 = s1
    mg.sample2 = s2
    mg.metrics[0].metricId = N.NVML_GPM_METRIC_DRAM_BW_UTIL
    mg.metrics[1].metricId = N.NVML_GPM_METRIC_SM_UTIL
    N.nvmlGpmMetricsGet(mg)
    util = mg.metrics[0].value
    moved = reps * 2 * a.numel() * 2
    print(f"reps {reps}: {moved / dt / 1e9:.0f} GB/s wall, DRAM_BW_UTIL {util:.1f}%, SM_UTIL {mg.metrics[1].value:.1f}%, "
          f"implied peak {moved / dt / 1e9 / (util / 100):.0f} GB/s")
