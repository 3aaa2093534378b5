"""H2D bandwidth from pinned host memory allocated under each NUMA node's CPU affinity
(first-touch places the pinned pages on the allocating thread's node).  Prints the GPU's own
NUMA node, so bench.py / SnpBatchStream can allocate their pinned rows next to the GPU."""
import glob
import os
import time

import torch


def cpulist(s):
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out


def gpu_numa_node():
    bdf = None   # torch's pci_bus_id is the bus number only: ask nvidia-smi for the full address
    if bdf is None:
        import subprocess
        bdf = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", "0"],
                             capture_output=True, text=True).stdout.strip()
    bdf = bdf.lower()
    if len(bdf.split(":")[0]) == 8:
        bdf = bdf[4:]
    p = f"/sys/bus/pci/devices/{bdf}/numa_node"
    return (open(p).read().strip() if os.path.exists(p) else "?"), bdf


def main():
    torch.cuda.init()
    print("gpu numa node / bdf:", gpu_numa_node())
    nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
    print("nodes:", len(nodes), "cpus allowed:", len(os.sched_getaffinity(0)))
    all_cpus = os.sched_getaffinity(0)
    nbytes = 1 << 30
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for nd in nodes:
        cpus = set(cpulist(open(nd + "/cpulist").read())) & all_cpus
        if not cpus:
            print(os.path.basename(nd), "no allowed cpus")
            continue
        os.sched_setaffinity(0, cpus)
        src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        src.fill_(1)
        for chunk in (nbytes, 51 << 20):
            best = 0.0
            for _ in range(4):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for off in range(0, nbytes - chunk + 1, chunk):
                    dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                n = (nbytes // chunk) * chunk
                best = max(best, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            print(os.path.basename(nd), f"cpus {min(cpus)}-{max(cpus)} chunk {chunk >> 20} MiB: {best:.1f} GB/s")
        # D2H too
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        src.copy_(dst, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        print(os.path.basename(nd), f"d2h {nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
        del src
        os.sched_setaffinity(0, all_cpus)


if __name__ == "__main__":
    main()
