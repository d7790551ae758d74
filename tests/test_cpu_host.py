"""CPU tests of the host side: the C ABI library loads and exports every declared symbol, the
product path refuses to run without a B200 (no CPU fallback), request sharding + the final gather
over a 2-rank gloo group, reference error conventions, and the CPU oracle's lossless-greedy
identity on the tiny config."""

import ctypes
import os
import re
import socket
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    from paper_2512_23858_b200 import _lib

    hdr = (ROOT / "include" / "ygg.h").read_text()
    declared = set(re.findall(r"\b(ygg_[a-z0-9_]+)\s*\(", hdr))
    raw = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in sorted(declared) if not hasattr(raw, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= declared, set(_lib.EXPORTED) - declared
    lib = _lib.load()
    assert lib.ygg_version() >= 100


def test_abi_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the C structs have the header's sizes and field offsets (compiled with gcc)."""
    import subprocess

    from paper_2512_23858_b200 import _lib

    structs = {"ygg_tree": _lib.YggTree, "ygg_seq": _lib.YggSeq, "ygg_profile": _lib.YggProfile,
               "ygg_profile_pair": _lib.YggProfilePair, "ygg_prune_args": _lib.YggPruneArgs,
               "ygg_epilogue": _lib.YggEpilogue, "ygg_gemv_epilogue": _lib.YggGemvEpilogue,
               "ygg_l2_region": _lib.YggL2Region}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ygg.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_argument_errors_map_to_value_error_without_device():
    """Host-side argument validation runs before any device work."""
    from paper_2512_23858_b200 import _lib

    lib = _lib.load()
    with pytest.raises(ValueError):
        _lib.check(lib.ygg_topk_softmax(None, 0, 1, 10, 10, 0, 1.0, None, None, None, None, 0, None))
    with pytest.raises(ValueError):
        _lib.check(lib.ygg_gemm_plan_init(ctypes.create_string_buffer(4096), 1, 1, 1, 1, 100, 64, 0, 1, None, None))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    from paper_2512_23858_b200 import _lib
    from paper_2512_23858_b200.engine import SpecDecoder, StepShape
    from paper_2512_23858_b200.model import init_weights, preset

    tc = preset("tiny-target")
    w = init_weights(tc, 0, torch.float32)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.require_device()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        SpecDecoder(tc, w, tc, w, StepShape(2, 2))


def test_shard_requests_partition():
    from paper_2512_23858_b200.dist import shard_requests

    for n in (0, 1, 7, 16, 64):
        for world in (1, 2, 4, 8):
            ids = [i for r in range(world) for i in shard_requests(n, world, r)]
            assert ids == list(range(n))
            sizes = [len(shard_requests(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_requests(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_req, out_q):
    import torch.distributed as dist

    from oracle.llama_ref import RefLlama, greedy_ar
    from paper_2512_23858_b200.dist import gather_generated, shard_requests
    from paper_2512_23858_b200.model import init_weights, preset

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = preset("tiny-target", n_layers=1)
    model = RefLlama(cfg, init_weights(cfg, 0, torch.float32))
    mine = {}
    for rid in shard_requests(n_req, world, rank):
        g = torch.Generator().manual_seed(1000 + rid)
        prompt = torch.randint(0, cfg.vocab, (8,), generator=g).tolist()
        mine[rid] = greedy_ar(model, prompt, 4, 32)
    merged = gather_generated(mine, world)
    if rank == 0:
        out_q.put(merged)
    dist.destroy_process_group()


def test_request_sharding_gather_gloo_world2():
    """Two ranks each decode their shard; the gathered result equals the single-process run."""
    import torch.multiprocessing as mp

    from oracle.llama_ref import RefLlama, greedy_ar
    from paper_2512_23858_b200.model import init_weights, preset

    n_req = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_req, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = preset("tiny-target", n_layers=1)
    model = RefLlama(cfg, init_weights(cfg, 0, torch.float32))
    for rid in range(n_req):
        g = torch.Generator().manual_seed(1000 + rid)
        prompt = torch.randint(0, cfg.vocab, (8,), generator=g).tolist()
        assert merged[rid] == greedy_ar(model, prompt, 4, 32)


def test_oracle_spec_decoding_is_lossless_greedy():
    """CPU oracle: EGT speculative decoding == plain greedy AR (tiny cfg1, coupled and independent)."""
    from oracle.llama_ref import RefLlama, greedy_ar
    from oracle.spec_ref import RefSpecDecoder
    from oracle.tree_ref import Profile
    from paper_2512_23858_b200.model import Coupling, init_weights, preset

    tc, dc = preset("tiny-target"), preset("tiny-draft")
    for cp in (None, Coupling(rank=256, logit_scale=8.0, head_noise=2.0, layer_gain=2.0)):
        tw, dw = init_weights(tc, 0, torch.float32, "cpu", cp), init_weights(dc, 1, torch.float32, "cpu", cp)
        prompt = torch.randint(0, tc.vocab, (16,), generator=torch.Generator().manual_seed(5)).tolist()
        ar = greedy_ar(RefLlama(tc, tw), prompt, 24, 96)
        sd = RefSpecDecoder(RefLlama(tc, tw), RefLlama(dc, dw), 4, 4, 8, 64, Profile(((1, 20.0), (64, 30.0))),
                            Profile(((1, 100.0), (64, 100.0))), 96)
        assert sd.generate(prompt, 24) == ar


def test_host_latency_errors_follow_reference():
    from paper_2512_23858_b200.latency import ConfigError, LatencyProfile, TreeShape, latency_at, load_profile

    with pytest.raises(ValueError):
        LatencyProfile(((1, 1.0),), "verifier")
    with pytest.raises(ValueError):
        LatencyProfile(((4, 1.0), (2, 2.0)), "verifier")
    with pytest.raises(ValueError):
        latency_at(LatencyProfile(((1, 1.0), (4, 2.0)), "drafter"), 0)
    with pytest.raises(ValueError):
        TreeShape(2, 2, 6)
    with pytest.raises(ConfigError):
        load_profile("/nonexistent.csv", "drafter")


def test_profiler_csv_round_trip(tmp_path):
    """K8 exports use the reference's on-disk formats (latency.py:164-190, scheduler.py:82-103):
    what the profiler writes, the reference-named loaders read back exactly."""
    from paper_2512_23858_b200.latency import latency_at, load_profile
    from paper_2512_23858_b200.profiler import write_profile_csv, write_stage_csv
    from paper_2512_23858_b200.scheduler import StageProfiles

    bps = [(1, 1093.31), (8, 1103.4), (64, 4452.74)]
    write_profile_csv(bps, tmp_path / "verify.csv")
    prof = load_profile(tmp_path / "verify.csv", "verifier")
    assert [latency_at(prof, w) for w, _ in bps] == [us for _, us in bps]
    rows = [("Verify", "base", 4452.74), ("Accept", "base", 296.94), ("HeadDraft", "base", 2195.0),
            ("DraftStep", "base", 1104.45)]
    write_stage_csv(rows, tmp_path / "stages.csv")
    sp = StageProfiles.from_csv(tmp_path / "stages.csv")
    for name, _, us in rows:
        assert sp.base(name) == us
    assert sp.base("DraftStep3") == 1104.45  # DraftStep fallback (reference scheduler.py:112-118)


def test_launcher_runs_world2_gloo(tmp_path):
    """dist.launch (what `bench.py --gpus N` uses when WORLD_SIZE is unset) starts N ranks under
    torch.distributed.run on 127.0.0.1; the gathered ids equal the single-process decode."""
    import json

    from oracle.llama_ref import RefLlama, greedy_ar
    from paper_2512_23858_b200.dist import launch
    from paper_2512_23858_b200.model import init_weights, preset

    out = tmp_path / "gathered.json"
    rc = launch(2, str(ROOT / "tests" / "_launch_worker.py"), [str(out), "5"], timeout=300)
    assert rc == 0
    got = json.loads(out.read_text())
    assert got["world"] == 2
    cfg = preset("tiny-target", n_layers=1)
    model = RefLlama(cfg, init_weights(cfg, 0, torch.float32))
    for rid in range(5):
        g = torch.Generator().manual_seed(1000 + rid)
        assert got["merged"][str(rid)] == greedy_ar(model, torch.randint(0, cfg.vocab, (8,), generator=g).tolist(), 4, 32)


def test_measured_b200_bundle_feeds_reference_offline_drivers():
    """§8 f2: the K8-measured B200 profiles (profiles/b200_cfg2, written by `bench.py --workload cfg3
    --export-profiles`) are in the reference's on-disk formats: our loaders read them, and — when the
    reference is installed in baseline/_ref — its own simulator reproduces the committed offline run."""
    import json

    from paper_2512_23858_b200.latency import latency_at, load_profile
    from paper_2512_23858_b200.scheduler import StageProfiles

    b = ROOT / "profiles" / "b200_cfg2"
    d = load_profile(b / "draft_profile.csv", "drafter")
    v = load_profile(b / "verify_profile.csv", "verifier")
    assert latency_at(v, 1) > 1000.0 and latency_at(d, 8) < latency_at(v, 1)
    sp = StageProfiles.from_csv(b / "stages.csv")
    assert sp.base("Verify") > 0 and sp.base("DraftStep5") == sp.base("DraftStep")
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "specsim").exists():
        pytest.skip("reference not installed in baseline/_ref")
    import importlib.util
    import sys

    spec = importlib.util.spec_from_file_location("reference_offline", ROOT / "scripts" / "reference_offline.py")
    mod = importlib.util.module_from_spec(spec)
    sys.path.insert(0, str(ref))
    spec.loader.exec_module(mod)
    got = mod.main(str(b))
    want = json.loads((b / "reference_offline.json").read_text())
    assert got["run"] == want["run"]
    assert [r["speedup"] for r in got["breakdown"]] == [r["speedup"] for r in want["breakdown"]]
