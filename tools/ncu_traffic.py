"""DRAM traffic of bench.py's roofline kernel from one ncu --set full capture.

    # on the GPU box: launch the kernel under ncu (one capture)
    ncu --set full --clock-control none -k regex:gemm_sk_kernel -s 6 -c 1 \
        -o gpurun_out/rNN_roofline python tools/ncu_traffic.py run
    # here: write profiles/rNN_ncu_traffic.json from the report
    python tools/ncu_traffic.py parse gpurun_out/rNN_roofline.ncu-rep profiles/rNN_ncu_traffic.json

`run` launches the verify gate/up GEMM (SiLU epilogue) at the bench shape, M =
m (k + 1) = 192, N = 28672, K = 4096, exactly as bench.py's roofline timing does
(stream-K, all SMs, rotating weights).  `parse` stores
dram__bytes_read.sum / dram__bytes_write.sum of the captured launch under the
key bench.py looks up.
"""
import csv
import json
import subprocess
import sys

M, N, K = 192, 28672, 4096


def run():
    import torch
    sys.path.insert(0, ".")
    from paper_2603_18016_b200 import native, ops
    dev = torch.device("cuda:0")
    ws = [torch.randn(N, K, device=dev).mul_(0.02).to(torch.bfloat16) for _ in range(4)]
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    out = torch.empty(M, N // 2, dtype=torch.bfloat16, device=dev)
    scratch = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    for i in range(10):
        ops.gemm(x, ws[i % 4], out=out, epi=native.EPI_SILU, workspace=scratch)
    torch.cuda.synchronize()
    print("done")


def parse(rep, out_json):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    d = dict(zip(hdr, rows[2]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    units = dict(zip(hdr, rows[1]))

    def val(k):
        return int(float(d[k].replace(",", "")) * scale.get(units[k], 1))
    res = {f"gate_up_M{M}_N{N}_K{K}": {
        "kernel": d["Kernel Name"][:120],
        "dram_read": val("dram__bytes_read.sum"),
        "dram_write": val("dram__bytes_write.sum"),
        "duration_us": float(d["gpu__time_duration.sum"].replace(",", "")) *
        {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}[units["gpu__time_duration.sum"]],
        "algorithmic_bytes": 2 * N * K + 2 * M * K + 2 * M * (N // 2),
        "source": f"ncu --set full --clock-control none, {rep}"}}
    with open(out_json, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2], sys.argv[3])
