"""tilefabric-bench on the B200 kernels: the reference CLI's own checks
(proj/tests/cli_test.cpp), flag handling and exit codes on CPU, the runs on
the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CLI_DIR = os.path.join(ROOT, "paper_2511_02168_b200", "cli")
BIN = os.path.join(CLI_DIR, "tilefabric-bench")


def run_bench(args):
    if not os.path.exists(BIN):
        subprocess.run(["make", "-s", "-C", CLI_DIR], check=True)
    r = subprocess.run([BIN] + args.split(), capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout + r.stderr, r.stdout


def split_csv(line):
    return line.split(",")


# ---- flag handling and exit codes (cli_test.cpp:110-159), no GPU needed ----

def test_help_exits_zero():
    code, out, _ = run_bench("--help")
    assert code == 0 and "--pattern" in out and "--world-size" in out


def test_unknown_flag_exits_two():
    code, out, _ = run_bench("--no-such-flag")
    assert code == 2 and "--help" in out


def test_unknown_pattern_exits_two():
    code, out, _ = run_bench("--pattern warp-drive")
    assert code == 2 and "warp-drive" in out and "ag-pull" in out


def test_missing_pattern_exits_two():
    assert run_bench("--world-size 2")[0] == 2


def test_non_divisible_shard_exits_two():
    code, out, _ = run_bench("--pattern fd-fused --world-size 3 --kv-len 64")
    assert code == 2 and "divisible" in out


def test_mixed_families_exit_two():
    assert run_bench("--patterns ag-pull,fd-bsp --world-size 2 --iters 1 --warmup 0")[0] == 2


def test_bad_skew_spec_exits_two():
    assert run_bench("--pattern ag-pull --skew nonsense --iters 1")[0] == 2
    assert run_bench("--pattern ag-pull --skew 0:-5 --iters 1")[0] == 2
    assert run_bench("--pattern ag-pull --skew 9:5 --world-size 2 --iters 1")[0] == 2


def test_zero_iters_exits_two():
    assert run_bench("--pattern ag-pull --iters 0")[0] == 2


def test_paper_fd_dry_run_echoes_the_configuration():
    code, out, _ = run_bench("--preset paper-fd --dry-run")
    assert code == 0
    for s in ("world_size: 8", "heads: 96", "head_dim: 128", "fd-fused"):
        assert s in out, out


def test_unknown_preset_exits_two():
    code, out, _ = run_bench("--preset desk-everything --dry-run")
    assert code == 2 and "desk-fd" in out


def test_explicit_flags_override_preset():
    code, out, _ = run_bench("--preset paper-fd --world-size 2 --dry-run")
    assert code == 0 and "world_size: 2" in out and "heads: 96" in out


def test_paper_ag_preset_sweeps_m():
    code, out, _ = run_bench("--preset paper-ag-gemm --dry-run")
    assert code == 0 and "n: 28672" in out and "k: 8192" in out and "m: 1 2 4" in out


# ---- runs on the GPU (cli_test.cpp:163-321) ----

@pytest.mark.gpu
def test_verified_single_run_exits_zero():
    code, out, stdout = run_bench("--pattern ag-pull --world-size 2 --m 8 --n 8 --k 8 --verify "
                                  "--iters 1 --warmup 0 --launch-cost-us 0")
    assert code == 0, out
    j = json.loads(stdout)
    assert j["pattern"] == "ag-pull" and j["verified"] is True
    assert j["max_error"] == 0.0  # config 1: bitwise
    assert j["latency_ms"]["median"] > 0.0
    assert j["taxes"]["staged_bytes"] == 0


@pytest.mark.gpu
def test_single_run_writes_iteration_csv_and_summary_json(tmp_path):
    prefix = str(tmp_path / "run")
    code, out, _ = run_bench("--pattern fd-fused --world-size 2 --heads 2 --head-dim 4 --kv-len 64 "
                             "--iters 5 --warmup 1 --launch-cost-us 0 --verify --out " + prefix)
    assert code == 0, out
    lines = open(prefix + ".csv").read().splitlines()
    assert len(lines) == 6
    assert "pattern,world_size" in lines[0] and "makespan_ms" in lines[0]
    ncol = len(split_csv(lines[0]))
    for i, line in enumerate(lines[1:]):
        cols = split_csv(line)
        assert len(cols) == ncol, line
        assert cols[0] == "fd-fused" and cols[1] == "2" and cols[2] == ""
        assert cols[5] == "2" and cols[6] == "4" and cols[7] == "64"
        assert cols[9] == str(i) and cols[15] == "true"
    j = json.load(open(prefix + ".json"))
    assert j["kv_len"] == 64 and j["iters"] == 5


@pytest.mark.gpu
def test_straggler_flag_feeds_the_taxes():
    # Rank 1 absorbs rank 0's 40 ms straggle in barrier waits (fd-bsp).
    code, out, stdout = run_bench("--pattern fd-bsp --world-size 2 --heads 1 --head-dim 4 --kv-len 8 "
                                  "--skew 0:40 --iters 1 --warmup 0 --launch-cost-us 0")
    assert code == 0, out
    assert json.loads(stdout)["taxes"]["bulk_sync_tax_ms"] >= 30.0
    # The fused schedule has no barrier to pay at: rank 1 waits on source 0.
    code, out, stdout = run_bench("--pattern fd-fused --world-size 2 --heads 1 --head-dim 4 --kv-len 8 "
                                  "--skew 0:40 --iters 1 --warmup 0 --launch-cost-us 0")
    assert code == 0, out
    j = json.loads(stdout)
    assert j["taxes"]["bulk_sync_tax_ms"] == 0.0 and j["taxes"]["wait_idle_ms"] >= 30.0


@pytest.mark.gpu
def test_fd_sweep_emits_one_verified_row_per_cell(tmp_path):
    prefix = str(tmp_path / "sweep")
    code, out, _ = run_bench("--patterns fd-bsp,fd-ag,fd-wait,fd-fused --sweep-kv 64,128,256 --world-size 4 "
                             "--heads 2 --head-dim 4 --iters 1 --warmup 0 --launch-cost-us 0 --verify --out "
                             + prefix)
    assert code == 0, out
    lines = open(prefix + ".csv").read().splitlines()
    assert len(lines) == 13 and "speedup_vs_baseline" in lines[0]
    ncol = len(split_csv(lines[0]))
    for line in lines[1:]:
        cols = split_csv(line)
        assert len(cols) == ncol, line
        assert cols[5] == "2" and cols[17] == "true" and float(cols[18]) > 0.0 and cols[19] == ""
    rows = [ln for ln in open(prefix + ".dat").read().splitlines() if ln and not ln.startswith("#")]
    assert len(rows) == 3
    for row in rows:
        assert len(row.split()) == 5


@pytest.mark.gpu
def test_ag_sweep_speedup_is_relative_to_baseline(tmp_path):
    prefix = str(tmp_path / "ag")
    code, out, _ = run_bench("--patterns ag-baseline,ag-pull --sweep-m 4,8 --world-size 2 --n 8 --k 8 "
                             "--iters 3 --warmup 0 --launch-cost-us 0 --out " + prefix)
    assert code == 0, out
    lines = open(prefix + ".csv").read().splitlines()
    assert len(lines) == 5
    for line in lines[1:]:
        cols = split_csv(line)
        assert cols[18] != ""
        if cols[0] == "ag-baseline":
            assert float(cols[18]) == 1.0
        else:
            assert float(cols[18]) > 0.0


@pytest.mark.gpu
def test_sweep_without_out_still_prints_rows():
    code, out, _ = run_bench("--patterns fd-bsp,fd-fused --world-size 2 --heads 1 --head-dim 4 --kv-len 16 "
                             "--iters 1 --warmup 0 --launch-cost-us 0")
    assert code == 0, out
    assert "fd-bsp,2," in out and "fd-fused,2," in out


@pytest.mark.gpu
def test_bf16_gqa_decode_and_gemm_verify():
    # GPU extensions: the tensor-core paths through the same CLI.
    code, out, stdout = run_bench("--pattern fd-fused --world-size 2 --batch 2 --heads 16 --kv-heads 2 "
                                  "--head-dim 128 --kv-len 4096 --dtype bf16 --verify --iters 3 --warmup 1")
    assert code == 0, out
    assert json.loads(stdout)["verified"] is True
    code, out, stdout = run_bench("--pattern ag-push --world-size 2 --m 256 --n 512 --k 512 --dtype bf16 "
                                  "--verify --iters 3 --warmup 1")
    assert code == 0, out
    assert json.loads(stdout)["verified"] is True
