import sys, time, torch
sys.path.insert(0, ".")  # run from the repo root
import bench
c = bench.ClockSampler(1); print("buses", c.buses); p = torch.cuda.get_device_properties(0); print(repr(p.uuid), type(p.uuid), getattr(p, "pci_bus_id", None), getattr(p, "pci_device_id", None), getattr(p, "pci_domain_id", None))
import subprocess; print(subprocess.run(["nvidia-smi", "--query-gpu=uuid,pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout)
c.start(); x = torch.randn(8192, 8192, device="cuda")
t = time.time()
while time.time() - t < 3: x = x @ x; x /= x.norm()
torch.cuda.synchronize(); print(c.stop())
