# PCIe copy-engine throughput vs copy size / direction / host DRAM load
mkdir -p gpurun_out
timeout 900 python tools/pcie_chunk_probe.py > gpurun_out/r2v_pcie_chunks.jsonl 2> gpurun_out/r2v_pcie_chunks.err
