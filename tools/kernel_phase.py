"""Bench phase name of a kernel launch (kernel template arguments + grid), shared by the
profile tools."""


# phase of a launch: kernel template kind + grid
def phase_of(name, grid):
    if name.startswith("k_interp"):
        return "interp_evolve"
    if name.startswith("k_force"):
        return "force"
    if name.startswith("k_spread") or name.startswith("k_brick"):
        return "spread"
    if name.startswith("k_xwarp"):
        # k_xwarp<L, KIND, DIM, NC, WPB, MINB>: x-line passes
        args = [a.strip() for a in name[name.index("<") + 1:name.index(">")].split(",")]
        return "s1_rhs_xsweep" if int(args[1]) == 0 else "psi_x_p"
    if name.startswith("k_lines") or name.startswith("k_strided"):
        # k_lines<L, KIND, DIM, AX, ...>, k_strided<L, KIND, DIM, AX>
        args = [a.strip() for a in name[name.index("<") + 1:name.index(">")].split(",")]
        kind, ax = int(args[1]), int(args[3])
        if kind == 0:
            return "s1_rhs_xsweep"
        if kind == 1:
            z = grid.split(",")[-1].strip(" )") if grid else "1"
            return "sweep_y" if z != "1" else "psi_y"
        if kind == 2:
            return "sweep_z" if ax == 2 else "sweep_y"
        if kind == 3:
            return "div_psi_first"
        if kind == 4:
            return "psi_x_p"
    return name
