"""Pretty-print tools/ncu_points.py output (one row per point)."""
import json
import sys

for l in open(sys.argv[1]):
    r = json.loads(l)
    g = lambda p: [v for k, v in r.items() if k.startswith(p)][0]  # noqa: E731
    M = 2 ** 27
    print(r['K'], r['C'], r['mode'], r['threads'], r['I'], "G/s %.1f" % r['G_lookups_per_s_under_ncu'],
          "dramB %.0f" % r['dram_B_per_lookup'], "GBps %.0f" % r['dram_GBps'], "inst %.1f" % r.get('inst_per_lookup', 0),
          "l1wf%% %.0f" % g('l1tex__data_pipe_lsu_wavefronts.avg.pct'), "wf/l %.1f" % (g('l1tex__data_pipe_lsu_wavefronts.sum') / M),
          "smwf/l %.1f" % (g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum') / M),
          "conf/l %.1f" % (g('l1tex__data_bank_conflicts') / M), "l2hit %.0f" % g('lts__t_sector_hit_rate'),
          "lts%% %.0f" % g('lts__throughput'), "regs", g('launch__registers'), "ipc %.2f" % g('sm__inst_executed.avg.per_cycle'),
          "fab/l %.1f" % (g('lts__t_requests_srcunit_ltcfabric') / M))
