"""Per-CTA %globaltimer timeline of one fused GEMM launch (debug stamps), for 1B/8B shapes."""
import ctypes as C, json, math, sys
import torch
sys.path.insert(0, ".")
from paper_2512_23858_b200 import _lib as L
from paper_2512_23858_b200.forward import GemmPlan
L.require_device(); lib = L.lib()
out = {}
for name, (N, K, M, kind) in {"1b.gu": (16384, 2048, 8, L.YGG_EPI_SWIGLU), "1b.down": (2048, 8192, 8, L.YGG_EPI_RESID),
                              "1b.qkv_none": (3072, 2048, 8, L.YGG_EPI_NONE), "8b.qkv": (6144, 4096, 50, L.YGG_EPI_SWIGLU),
                              "8b.gu": (28672, 4096, 50, L.YGG_EPI_SWIGLU)}.items():
    W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    plan = GemmPlan(W, X, M)
    ws = torch.zeros(plan.ws_bytes // 4 + 16, device="cuda")
    cnt = torch.zeros(plan.tiles, dtype=torch.int32, device="cuda")
    dbg = torch.zeros(160, 8, dtype=torch.int64, device="cuda")
    act = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    resid = torch.zeros(M, N, device="cuda"); hb = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    ss = torch.zeros(N // 128, M, device="cuda")
    e = L.YggEpilogue(); e.kind = kind; e.counters = cnt.data_ptr(); e.dbg = dbg.data_ptr()
    e.act_out = act.data_ptr(); e.resid = resid.data_ptr(); e.hb = hb.data_ptr(); e.ss_out = ss.data_ptr()
    for it in range(4):
        dbg.zero_()
        L.check(lib.ygg_gemm_fused(plan.handle, ws.data_ptr(), C.byref(e), L.stream_ptr()))
        torch.cuda.synchronize()
    d = dbg.cpu()
    n = (d[:, 0] > 0).sum().item()
    d = d[:n].double()
    t0 = d[:, 0].min()
    rel = (d - t0) / 1000.0
    rel[d == 0] = float('nan')
    cols = ["start", "epi_loop_end", "fix0_go", "fix1_go", "fix_end", "mma_end", "prod_end"]
    stats = {c: [round(float(torch.nanmean(rel[:, i])), 2), round(float(rel[:, i][~torch.isnan(rel[:, i])].max()) if (~torch.isnan(rel[:, i])).any() else -1, 2)] for i, c in enumerate(cols)}
    out[name] = {"ctas": n, "segments": plan.segments, "tiles": plan.tiles, "mean_max_us": stats}
    print(name, json.dumps(out[name]), flush=True)
