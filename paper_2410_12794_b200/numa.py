"""Host NUMA placement for the host-buffer (e2e) path.

Pinned host buffers are placed on the NUMA node of the thread that
allocates them. On multi-socket GPU boxes a buffer on the far socket sends
every H2D/D2H copy across the inter-socket link, which caps the host API
below the PCIe rate. `bind_to_device` restricts the calling process to the
CPUs the GPU's PCIe root reports as local (sysfs `local_cpulist`), so the
pinned staging buffers allocated afterwards sit next to the GPU.
"""

from __future__ import annotations

import os


def _parse_cpulist(text: str) -> list:
    cpus = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            lo, hi = part.split("-")
            cpus.extend(range(int(lo), int(hi) + 1))
        else:
            cpus.append(int(part))
    return cpus


def device_local_cpus(device=0) -> list:
    """CPUs local to `device`'s PCIe attachment ([] when sysfs has no answer)."""
    import torch
    p = torch.cuda.get_device_properties(device)
    path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0/local_cpulist"
    try:
        with open(path) as fh:
            cpus = _parse_cpulist(fh.read())
    except OSError:
        return []
    allowed = os.sched_getaffinity(0)
    return [c for c in cpus if c in allowed]


def bind_to_device(device=0) -> list:
    """Restrict this process to `device`'s local CPUs; returns them ([] = unchanged)."""
    cpus = device_local_cpus(device)
    if cpus and set(cpus) != os.sched_getaffinity(0):
        os.sched_setaffinity(0, cpus)
        return cpus
    return []
