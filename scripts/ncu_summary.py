"""Summarise an ncu raw-page CSV (ncu -i X.ncu-rep --page raw --csv) into a small per-launch table."""
import csv
import sys

KEEP = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__sass_thread_inst_executed_op_ffma_pred_on.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active',
        'lts__t_bytes.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'launch__shared_mem_per_block_dynamic', 'launch__occupancy_limit_registers']


def main(src, dst):
    r = list(csv.reader(open(src)))
    h, u, rows = r[0], r[1], r[2:]
    with open(dst, 'w', newline='') as f:
        w = csv.writer(f)
        w.writerow(['metric', 'unit'] + [f'launch{i}' for i in range(len(rows))])
        stalls = [k for k in h if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio')]
        for k in KEEP + stalls:
            if k in h:
                i = h.index(k)
                w.writerow([k, u[i]] + [row[i] for row in rows])


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])
