"""FP64 pipe vs FP64 tensor core (DMMA m8n8k4) throughput on this GPU:
mode 0 DFMA, 1 DMMA, 2 both interleaved (ldg_probe_fp64_mode)."""
import ctypes, json, sys
sys.path.insert(0, ".")
from paper_2205_07824_b200._lib import load, check
lib = load()
out = {}
for mode, name in ((0, "dfma"), (1, "dmma"), (2, "dfma+dmma")):
    tf, ms = ctypes.c_double(), ctypes.c_double()
    check(lib.ldg_probe_fp64_mode(mode, 20000, ctypes.byref(tf), ctypes.byref(ms), None), "probe")
    out[name] = {"tflops": tf.value, "ms": ms.value}
print(json.dumps(out))
