"""Summarise an ncu --set full report of one tab_round launch (development tool):
duration, pipe utilisation, instructions / POPC per codeword, DRAM bytes, stall mix."""
import csv
import io
import subprocess
import sys


SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
         "nsecond": 1e-9, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}


def raw(rep):
    """metric -> value in base units (seconds, bytes) using the report's unit row; `rep` is an
    .ncu-rep or a saved `ncu -i REP --page raw --csv` page"""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = {}
    for name, unit, val in zip(rows[0], rows[1], rows[2]):
        try:
            d[name] = float(val.replace(",", "")) * SCALE.get(unit, 1.0)
        except ValueError:
            d[name] = val
    return d


def main(rep, codewords):
    d = raw(rep)
    f = lambda k: d[k] if isinstance(d.get(k), float) else float("nan")
    dur_ns = f("gpu__time_duration.sum") * 1e9
    sms = f("device__attribute_multiprocessor_count")
    cyc = f("sm__cycles_active.avg")
    xu_pct = f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active")
    alu_pct = f("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")
    inst = f("smsp__inst_executed.sum")
    xu_ops = xu_pct / 100 * cyc * sms * 16  # 16 XU lanes/clk/SM
    alu_ops = alu_pct / 100 * cyc * sms * 64  # 64 ALU lanes/clk/SM (LOP3, IADD3, ISETP, IMNMX, ...)
    dram = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
    lines = [
        f"report: {rep}",
        f"kernel: {d.get('Kernel Name', '?')}",
        f"duration: {dur_ns / 1e3:.1f} us   codewords: {codewords}   codewords/s: {codewords / (dur_ns * 1e-9):.4e}",
        f"SM active cycles (avg): {cyc:.0f}   SMs: {sms:.0f}   grid: {d.get('launch__grid_size')}   regs/thread: {d.get('launch__registers_per_thread')}",
        f"XU (POPC) pipe busy while active: {xu_pct:.1f} %   ALU pipe busy while active: {alu_pct:.1f} %",
        f"warp instructions: {inst:.4e}   thread instructions per codeword: {inst * 32 / codewords:.2f}",
        f"XU ops per codeword: {xu_ops / codewords:.3f}   ALU-pipe ops per codeword: {alu_ops / codewords:.3f}",
        f"pipe-bound peak (SM-active clock): ALU {sms * 64 * cyc / (dur_ns * 1e-9) / (alu_ops / codewords):.4e} cw/s,"
        f" XU {sms * 16 * cyc / (dur_ns * 1e-9) / (xu_ops / codewords):.4e} cw/s",
        f"DRAM bytes (read + write): {dram:.0f}",
        f"achieved occupancy: {d.get('sm__warps_active.avg.pct_of_peak_sustained_active')} %",
    ]
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
