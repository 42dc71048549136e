"""Multi-rank paths on one B200 (two processes sharing cuda:0, gloo): the
sharded single-trace replay (replicated formation, jobs split
by first batch, MAX all_reduce of job results, SUM all_reduce of the owned
per-batch outputs) and the LPT-split C5 sweep with its gathered per-scenario
rows -- both bit-identical to the one-rank results."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _c4_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.distributed import replay_trace_sharded
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=2e5, seed=3)
    pipe = engine.ReplayPipeline([spec], t16.arrays(), scale=1.5)
    st = replay_trace_sharded(pipe, min_len=32, passes=2, backend="gloo")
    v = pipe.scenario(pipe.fetch(), 0)
    np.savez(os.path.join(out, f"c4_{rank}.npz"), **{k: np.asarray(v[k]) for k in
                                                      ("order", "b_start", "b_completion", "b_measured", "b_nseg",
                                                       "r_slo_met", "slo_n", "slo_met", "slo_p", "status",
                                                       "n_reseats", "n_segments")},
             rank_batches=np.array(st["rank_batches"]), jobs=np.array([st["jobs_initial"], st["jobs_final"]]))
    dist.destroy_process_group()


def test_sharded_single_trace_equals_one_rank():
    from paper_2512_18725_b200 import engine
    from paper_2512_18725_b200.sweep import c4_scenario, table16

    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_c4_worker, args=(world, _port(), out), nprocs=world, join=True)
        got = [dict(np.load(os.path.join(out, f"c4_{r}.npz"))) for r in range(world)]
    t16, arch = table16()
    spec = c4_scenario(t16, arch, n_requests=2e5, seed=3)
    pipe = engine.ReplayPipeline([spec], t16.arrays(), scale=1.5)
    engine.replay_segmented(pipe, min_len=32, passes=2)
    ref = pipe.scenario(pipe.fetch(), 0)
    # both ranks did a share of the trace, and each assembled the whole of it
    (a0, b0), (a1, b1) = got[0]["rank_batches"], got[1]["rank_batches"]
    assert a0 == 0 and b0 == a1 and b1 == len(ref["order"]) and 0 < a1 < b1
    for g in got:
        for k in ("order", "b_start", "b_completion", "b_measured", "b_nseg", "r_slo_met", "slo_n", "slo_met",
                  "slo_p"):
            assert np.array_equal(g[k], np.asarray(ref[k])), k
        assert int(g["status"]) == 0 and int(g["n_reseats"]) == ref["n_reseats"]
        assert int(g["n_segments"]) == ref["n_segments"]


def _c5_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.distributed import SweepRows, gather_sweep_rows, lpt_shards
    from paper_2512_18725_b200.sweep import c5_scenarios, expected_requests

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    table = p.gen_synthetic_profiles()
    specs = c5_scenarios(table, 300)
    shards = lpt_shards([expected_requests(s) for s in specs], world)
    preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
    pipe = engine.ReplayPipeline([specs[i] for i in shards[rank]], table.arrays(), preds=preds, scale=1.5,
                                 evaluate=(0, 1, 0.99))
    pipe.run()
    blocks = gather_sweep_rows(SweepRows(pipe).build(), [len(s) for s in shards], backend="gloo")
    rows = np.full((len(specs), blocks[0].shape[1]), np.nan)
    for r, blk in enumerate(blocks):
        rows[np.asarray(shards[r])] = blk.cpu().numpy()
    np.save(os.path.join(out, f"c5_{rank}.npy"), rows)
    dist.destroy_process_group()


def test_lpt_split_sweep_gathers_one_rank_rows():
    import paper_2512_18725_b200 as p
    from paper_2512_18725_b200 import _abi, engine
    from paper_2512_18725_b200.distributed import SweepRows
    from paper_2512_18725_b200.sweep import c5_scenarios

    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_c5_worker, args=(world, _port(), out), nprocs=world, join=True)
        got = [np.load(os.path.join(out, f"c5_{r}.npy")) for r in range(world)]
    table = p.gen_synthetic_profiles()
    preds = [_abi.Predictor(ewma=0, alpha=1.0, w=(0.0,) * 7), _abi.Predictor(ewma=1, alpha=0.5, w=(0.0,) * 7)]
    pipe = engine.ReplayPipeline(c5_scenarios(table, 300), table.arrays(), preds=preds, scale=1.5,
                                 evaluate=(0, 1, 0.99))
    pipe.run()
    ref = SweepRows(pipe).build().cpu().numpy()
    for g in got:
        np.testing.assert_array_equal(g, ref)
