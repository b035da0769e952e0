# e2e breakdown: the host-CSR build (gs_engine_load_csr from pinned host) vs the device-CSR build
python - <<'PY'
import ctypes, time, torch, sys
sys.path.insert(0, ".")
from fractions import Fraction
from paper_2311_12281_b200 import _lib
lib = _lib.load()
n = 1 << 24; cnt = 16 << 24
src = torch.empty(cnt, dtype=torch.int32, device="cuda"); dst = torch.empty_like(src)
_lib.check(lib.gs_rmat_generate(24, 16, 1, src.data_ptr(), dst.data_ptr(), None)); torch.cuda.synchronize()
uv = torch.empty(2 * cnt, dtype=torch.int32, device="cuda"); mm = ctypes.c_int64(0)
_lib.check(lib.gs_normalize_edges(cnt, src.data_ptr(), dst.data_ptr(), uv.data_ptr(), ctypes.byref(mm), None))
m = mm.value; del src, dst
off = torch.empty(n + 1, dtype=torch.int64, device="cuda"); adj = torch.empty(2 * m, dtype=torch.int32, device="cuda")
_lib.check(lib.gs_build_csr_device(n, m, uv.data_ptr(), off.data_ptr(), adj.data_ptr(), None)); torch.cuda.synchronize()
off_h = torch.empty(n + 1, dtype=torch.int64, pin_memory=True); adj_h = torch.empty(2 * m, dtype=torch.int32, pin_memory=True)
off_h.copy_(off); adj_h.copy_(adj)
eng = _lib.Engine(); eps2 = _lib.eps2_struct(Fraction("0.5"))
role = torch.empty(n, dtype=torch.uint8, pin_memory=True); clus = torch.empty(n, dtype=torch.int32, pin_memory=True)
st = _lib.GsStats()
# pure H2D of the same bytes
t = torch.empty(2 * m, dtype=torch.int32, device="cuda"); torch.cuda.synchronize()
t0 = time.perf_counter(); t.copy_(adj_h, non_blocking=True); off.copy_(off_h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"raw H2D of the CSR ({(8*(n+1)+8*m)/1e9:.2f} GB): {1e3*(t1-t0):.1f} ms")
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _lib.check(lib.gs_engine_load_csr(eng.handle, n, m, off_h.data_ptr(), adj_h.data_ptr(), 0))
    t1 = time.perf_counter()
    _lib.check(lib.gs_engine_scan(eng.handle, 5, ctypes.byref(eps2), role.data_ptr(), clus.data_ptr(), 0, ctypes.byref(st)))
    t2 = time.perf_counter()
    print(f"host-CSR load {1e3*(t1-t0):.1f} ms (build ev {st.phase_ms[1]:.1f}), scan {1e3*(t2-t1):.1f} ms (identify {st.phase_ms[2]:.1f} d2h {st.phase_ms[6]:.2f})")
PY
