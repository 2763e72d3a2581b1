"""Synthetic robot, scenes and plan skeletons for the five BASELINE.json configs.

Everything here is a PROPOSAL: the paper gives no robot
model, sphere model or scene geometry.  The robot is a Panda-like 7-DOF arm
described by public modified-DH numbers; the scenes mimic the *shapes* of the
paper's workloads (pick-place running example P:241-244, obstruction stacking
Fig. 2, Tetris packing P:810-813 with the min-object-distance goal cost
P:277-290 / P:769, trajectory knots Fig. 9).

Pure data: no forward kinematics, no costs, no sampling arithmetic.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np

# variable kinds (P:1006-1014 types conf/traj/grasp/placement)
CONF, PLACEMENT, GRASP, TRAJ = 0, 1, 2, 3
# action kinds (Listing 1; PressButton / PressButtonStick of the Stick Button domain)
MOVE_FREE, PICK, MOVE_HOLD, PLACE, PRESS, PRESS_STICK = 0, 1, 2, 3, 4, 5

INF = float("inf")


@dataclasses.dataclass
class Robot:
    """Serial 7-DOF arm, modified (Craig) DH: frame_j = frame_{j-1} * Rx(alpha) Tx(a) Tz(d) Rz(q_j).

    dh[j] = (a_{j-1}, d_j, alpha_{j-1}).  Tool (TCP) frame = frame_7 * Tz(flange_d) Rz(tcp_yaw) Tz(tcp_d).
    spheres[s] = (x, y, z, r) in the frame of link sphere_link[s] (1..7 = frame after joint j,
    8 = tool frame).  base = (x, y, z, yaw) of frame 0 in the world.
    """
    dh: np.ndarray            # (7, 3)
    flange_d: float
    tcp_yaw: float
    tcp_d: float
    joint_lo: np.ndarray      # (7,)
    joint_hi: np.ndarray      # (7,)
    spheres: np.ndarray       # (S, 4)
    sphere_link: np.ndarray   # (S,) int in 1..8
    base: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(4))
    # self-collision sphere pairs (i < j) checked by the SELF term
    self_pairs: List[tuple] = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class OBB:
    """Static oriented box: world pose and half extents.  Orientation: R (3x3 box-to-world rotation)
    if given, else Rz(yaw) about the world z axis."""
    center: np.ndarray        # (3,)
    yaw: float
    half: np.ndarray          # (3,)
    name: str = ""
    R: Optional[np.ndarray] = None   # (3, 3) full orientation; None = Rz(yaw)


@dataclasses.dataclass
class Obj:
    """Movable object approximated by spheres.  Object frame origin = bottom centre (L15)."""
    name: str
    spheres: np.ndarray       # (m, 4) object frame
    init_pose: np.ndarray     # (4,) x, y, z, yaw
    footprint: float          # radius used to shrink placement sampling regions
    grasp_xy: float           # top-down grasp sampler: TCP xy uniform in [-grasp_xy, grasp_xy]^2 (object frame)
    grasp_z: float            # TCP height above the object bottom
    grasp_mode: int = 0       # 0: top-down 4-DOF grasps; 1: 6-DOF grasps (top or one of the four sides)
    grasp_y: float = -1.0     # top-down grasp TCP y range (< 0: same as grasp_xy); e.g. along a stick


@dataclasses.dataclass
class Surface:
    """Placement surface: frame (x, y, z_top, yaw) in the world, rectangular region lo/hi in that frame.

    support_obb / support_obj name what the placed object rests on (excluded from CFreePlace, L3).
    """
    name: str
    frame: np.ndarray         # (4,) x, y, z_top, yaw
    lo: np.ndarray            # (2,)
    hi: np.ndarray            # (2,)
    support_obb: int = -1
    support_obj: int = -1


@dataclasses.dataclass
class Var:
    """Continuous skeleton parameter.  const=True marks the bold constants (q0, p0)."""
    kind: int
    name: str
    const: bool = False
    value: Optional[np.ndarray] = None    # constants: conf (7,) or placement (4,)
    obj: int = -1                         # grasp / placement: object
    surface: int = -1                     # placement: surface it is sampled on
    n_knots: int = 0                      # traj: free knots
    lo: Optional[np.ndarray] = None       # placement clamp bounds (4,) (L11)
    hi: Optional[np.ndarray] = None
    rng_stream: int = 0                   # sampler stream (Philox counter word); 0 = the variable's index


@dataclasses.dataclass
class Action:
    """Ground action of the skeleton (Listing 1).  Fields unused by a kind are -1."""
    kind: int
    obj: int = -1
    grasp: int = -1
    placement: int = -1
    surface: int = -1
    q1: int = -1
    q2: int = -1          # MoveFree/MoveHold target conf; Pick/Place use q1 as their conf
    traj: int = -1


@dataclasses.dataclass
class ProblemSpec:
    name: str
    robot: Robot
    obbs: List[OBB]
    objects: List[Obj]
    surfaces: List[Surface]
    variables: List[Var]
    actions: List[Action]
    goal_objs: List[int]
    # cost weights lambda_c and tolerances eps_c
    lam: dict
    eps: dict
    lam_goal: float = 0.025     # L7 (revised): the main-text Table 3 value
    lam_traj: float = 0.01      # L8, revised: 1.0 let the plan cost overpower the Kin constraints
    eta: float = 0.0            # collision activation distance (L1)
    # Adam (L9)
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    lr_conf: float = 0.01
    lr_pos: float = 0.005
    lr_yaw: float = 0.01
    lr_knot: float = 0.01
    self_collision: bool = False      # robot self-collision term per conf / knot
    collision_smooth: bool = False    # CHOMP-smooth collision cost (needs eta > 0)
    n_particles: int = 256
    n_steps: int = 100
    # conditional IK sampler in InitializeParticles: damped-least-squares iterations (0 = uniform
    # confs only, the paper's `Optimization` baseline init)
    ik_iters: int = 0
    ik_damping: float = 0.1
    ik_seeds: int = 1           # IK restarts per conf (R6): 1, 2, 4 or 8


DEFAULT_LAM = dict(JL=1.0, CF=1.0, KP=1.0, KR=5.0, SS=2.0, SC=2.0, CP=1.0, SELF=1.0, PC=1.0)
DEFAULT_EPS = dict(JL=0.0, CF=1e-3, KP=5e-3, KR=0.05, SS=1e-2, SC=1e-3, CP=1e-3, SELF=0.0, PC=1e-3)


def _line_spheres(p0, p1, r, n=4):
    p0 = np.asarray(p0, float)
    p1 = np.asarray(p1, float)
    return [list(p0 + (p1 - p0) * (k / (n - 1))) + [r] for k in range(n)]


def panda_robot() -> Robot:
    """Panda-like arm (public Franka modified-DH; NOT from the paper, L16)."""
    hp = math.pi / 2
    dh = np.array([
        [0.0, 0.333, 0.0],
        [0.0, 0.0, -hp],
        [0.0, 0.316, hp],
        [0.0825, 0.0, hp],
        [-0.0825, 0.384, -hp],
        [0.0, 0.0, hp],
        [0.088, 0.0, hp],
    ])
    lo = np.array([-2.8973, -1.7628, -2.8973, -3.0718, -2.8973, -0.0175, -2.8973])
    hi = np.array([2.8973, 1.7628, 2.8973, -0.0698, 2.8973, 3.7525, 2.8973])
    sph = []
    link = []

    def add(lst, l):
        for s in lst:
            sph.append(s)
            link.append(l)

    # 4 spheres per link, 8 links (7 DH links + tool frame) = 32 (S_r = 32, Appendix B)
    add(_line_spheres([0, 0, -0.19], [0, 0, -0.02], 0.07), 1)
    add(_line_spheres([0, -0.02, 0], [0, -0.26, 0.0], 0.07), 2)
    add(_line_spheres([0, 0, -0.10], [0.0825, 0, 0.0], 0.06), 3)
    add(_line_spheres([0, 0, 0], [-0.06, 0.12, 0.0], 0.06), 4)
    add(_line_spheres([0, 0.02, -0.27], [0, 0.06, -0.02], 0.055), 5)
    add(_line_spheres([0, 0, -0.01], [0.088, 0, -0.01], 0.05), 6)
    add(_line_spheres([0, 0, 0.02], [0.03, 0.03, 0.09], 0.045), 7)
    # tool frame (TCP, z = approach): hand + two finger pads
    add([[0, 0.05, -0.065, 0.03], [0, -0.05, -0.065, 0.03],
         [0, 0.042, -0.01, 0.012], [0, -0.042, -0.01, 0.012]], 8)
    # self-collision pairs: spheres on non-adjacent links, minus the structural overlap of the sphere model
    # (pair (7, 12) overlaps in 100 % of uniformly sampled confs; tools/gen_self_pairs.py)
    ignore = {(7, 12)}
    pairs = [(i, j) for i in range(len(sph)) for j in range(i + 1, len(sph))
             if abs(link[i] - link[j]) >= 2 and (i, j) not in ignore]
    return Robot(dh=dh, flange_d=0.107, tcp_yaw=-math.pi / 4, tcp_d=0.1034,
                 joint_lo=lo, joint_hi=hi, spheres=np.array(sph, float),
                 sphere_link=np.array(link, np.int32), self_pairs=pairs)


Q_HOME = np.array([0.0, -math.pi / 4, 0.0, -3 * math.pi / 4, 0.0, math.pi / 2, math.pi / 4])

TABLE = OBB(center=np.array([0.4, 0.0, -0.025]), yaw=0.0, half=np.array([0.7, 0.8, 0.025]), name="table")


def block(name, edge, pose, grasp_xy=0.005):
    """Cube of the given edge: 2x2x2 spheres (Appendix B)."""
    q = edge / 4
    sph = [[sx * q, sy * q, z, q] for z in (q, 3 * q) for sx in (-1, 1) for sy in (-1, 1)]
    return Obj(name=name, spheres=np.array(sph, float), init_pose=np.array(pose, float),
               footprint=edge / 2 * math.sqrt(2), grasp_xy=grasp_xy, grasp_z=min(0.6 * edge, 0.03))


def tall_block(name, edge, height, pose):
    """Tall box: 2x2 columns x 2 levels of spheres."""
    r = edge / 4
    sph = [[sx * r, sy * r, z, r] for z in (r, height - r) for sx in (-1, 1) for sy in (-1, 1)]
    return Obj(name=name, spheres=np.array(sph, float), init_pose=np.array(pose, float),
               footprint=edge / 2 * math.sqrt(2), grasp_xy=0.005, grasp_z=height - 0.025)


CELL = 0.04
TETROMINOES = {
    "I": [(0, 0), (1, 0), (2, 0), (3, 0)],
    "L": [(0, 0), (0, 1), (0, 2), (1, 0)],
    "J": [(1, 0), (1, 1), (1, 2), (0, 0)],
    "O": [(0, 0), (1, 0), (0, 1), (1, 1)],
}


def tetromino(name, shape, pose):
    """Four 4 cm cubes, two spheres per cube (S_o = 8; Appendix B)."""
    cells = np.array(TETROMINOES[shape], float) * CELL
    cells -= cells.mean(axis=0)
    r = 0.015
    sph = [[cx, cy, z, r] for cx, cy in cells for z in (0.015, 0.025)]
    ext = float(np.max(np.linalg.norm(cells, axis=1))) + CELL / 2
    return Obj(name=name, spheres=np.array(sph, float), init_pose=np.array(pose, float),
               footprint=ext, grasp_xy=0.005, grasp_z=0.025)


def _table_bounds():
    lo = np.array([TABLE.center[0] - TABLE.half[0], TABLE.center[1] - TABLE.half[1], -INF, -INF])
    hi = np.array([TABLE.center[0] + TABLE.half[0], TABLE.center[1] + TABLE.half[1], INF, INF])
    return lo, hi


class _Builder:
    """Tiny helper that appends variables/actions in skeleton order."""

    def __init__(self):
        self.vars: List[Var] = []
        self.actions: List[Action] = []

    def var(self, v: Var) -> int:
        self.vars.append(v)
        return len(self.vars) - 1

    def pick_place(self, obj: int, p0: int, surface: int, q_prev: int, tag: str, knots: int = 0):
        """MoveFree(q_prev, q_a) Pick(o, g, p0, q_a) MoveHold(o, g, q_a, q_b) Place(o, g, p1, s, q_b)."""
        lo, hi = _table_bounds()
        g = self.var(Var(GRASP, f"g_{tag}", obj=obj))
        qa = self.var(Var(CONF, f"q_pick_{tag}"))
        qb = self.var(Var(CONF, f"q_place_{tag}"))
        p1 = self.var(Var(PLACEMENT, f"p_{tag}", obj=obj, surface=surface, lo=lo, hi=hi))
        t1 = self.var(Var(TRAJ, f"tau_free_{tag}", n_knots=knots)) if knots else -1
        t2 = self.var(Var(TRAJ, f"tau_hold_{tag}", n_knots=knots)) if knots else -1
        self.actions.append(Action(MOVE_FREE, q1=q_prev, q2=qa, traj=t1))
        self.actions.append(Action(PICK, obj=obj, grasp=g, placement=p0, q1=qa))
        self.actions.append(Action(MOVE_HOLD, obj=obj, grasp=g, q1=qa, q2=qb, traj=t2))
        self.actions.append(Action(PLACE, obj=obj, grasp=g, placement=p1, surface=surface, q1=qb))
        return qb, p1


def _spec(name, objects, obbs, surfaces, b: _Builder, goal_objs, n, steps, **kw):
    return ProblemSpec(name=name, robot=panda_robot(), obbs=obbs, objects=objects, surfaces=surfaces,
                       variables=b.vars, actions=b.actions, goal_objs=goal_objs,
                       lam=dict(DEFAULT_LAM), eps=dict(DEFAULT_EPS), n_particles=n, n_steps=steps, **kw)


def config_pickplace(n=256, steps=100):
    """Config 1: the running example: one 5 cm block from the table into a 20x20 cm region."""
    objs = [block("red", 0.05, [0.45, -0.30, 0.0, 0.0])]
    obbs = [TABLE]
    surfs = [Surface("goal_region", np.array([0.55, 0.25, 0.0, 0.0]), np.array([-0.1, -0.1]),
                     np.array([0.1, 0.1]), support_obb=0)]
    b = _Builder()
    q0 = b.var(Var(CONF, "q0", const=True, value=Q_HOME.copy()))
    p0 = b.var(Var(PLACEMENT, "p0_red", const=True, value=objs[0].init_pose.copy(), obj=0))
    b.pick_place(0, p0, 0, q0, "red")
    return _spec("pickplace", objs, obbs, surfs, b, [], n, steps)


def config_obstruction(n=8192, steps=100):
    """Config 2: blue 8 cm block flanked by two tall obstructors; move both to a side region,
    then stack red on blue (Fig. 2).  3 pick-place actions."""
    blue_pose = [0.55, 0.05, 0.0, 0.0]
    objs = [
        block("blue", 0.08, blue_pose),
        tall_block("obsA", 0.05, 0.16, [0.55, 0.05 + 0.075, 0.0, 0.0]),
        tall_block("obsB", 0.05, 0.16, [0.55, 0.05 - 0.075, 0.0, 0.0]),
        block("red", 0.05, [0.40, -0.35, 0.0, 0.0]),
    ]
    obbs = [TABLE]
    surfs = [
        Surface("side_region", np.array([0.35, 0.40, 0.0, 0.0]), np.array([-0.1, -0.08]),
                np.array([0.1, 0.08]), support_obb=0),
        Surface("blue_top", np.array([blue_pose[0], blue_pose[1], 0.08, 0.0]), np.array([-0.04, -0.04]),
                np.array([0.04, 0.04]), support_obj=0),
    ]
    b = _Builder()
    q = b.var(Var(CONF, "q0", const=True, value=Q_HOME.copy()))
    p0s = [b.var(Var(PLACEMENT, f"p0_{o.name}", const=True, value=o.init_pose.copy(), obj=i))
           for i, o in enumerate(objs)]
    q, _ = b.pick_place(1, p0s[1], 0, q, "obsA")
    q, _ = b.pick_place(2, p0s[2], 0, q, "obsB")
    q, _ = b.pick_place(3, p0s[3], 1, q, "red")
    return _spec("obstruction", objs, obbs, surfs, b, [], n, steps)


def _tetris(n_pieces, shapes, region_cells, n, steps, goal, knots, name):
    cw, ch = region_cells
    slack = math.sqrt(1.15)                 # <= 15 % area slack
    rw, rh = cw * CELL * slack, ch * CELL * slack
    cx, cy = 0.50, 0.22
    wall_t, wall_h = 0.01, 0.06
    obbs = [TABLE,
            OBB(np.array([cx, cy + rh / 2 + wall_t / 2, wall_h / 2]), 0.0, np.array([rw / 2 + wall_t, wall_t / 2, wall_h / 2]), "wall_n"),
            OBB(np.array([cx, cy - rh / 2 - wall_t / 2, wall_h / 2]), 0.0, np.array([rw / 2 + wall_t, wall_t / 2, wall_h / 2]), "wall_s"),
            OBB(np.array([cx + rw / 2 + wall_t / 2, cy, wall_h / 2]), 0.0, np.array([wall_t / 2, rh / 2, wall_h / 2]), "wall_e"),
            OBB(np.array([cx - rw / 2 - wall_t / 2, cy, wall_h / 2]), 0.0, np.array([wall_t / 2, rh / 2, wall_h / 2]), "wall_w")]
    objs = []
    for i in range(n_pieces):
        row, col = divmod(i, 3)
        # Tetris-6: its second row starts 5 cm closer to the base, so that its last piece (at 0.81 m otherwise) is
        # within the arm's top-down reach (a top-down grasp at the old pose misses its Kin target by >= 5.09 mm,
        # the 5 mm tolerance of P:1133); Tetris-4's single piece in that row keeps its pose
        dx = -0.05 if (row and n_pieces > 4) else 0.0
        objs.append(tetromino(f"t{i}_{shapes[i]}", shapes[i], [0.30 + 0.17 * col + dx, -0.32 - 0.17 * row, 0.0, 0.0]))
    surfs = [Surface("tetris_region", np.array([cx, cy, 0.0, 0.0]), np.array([-rw / 2, -rh / 2]),
                     np.array([rw / 2, rh / 2]), support_obb=0)]
    b = _Builder()
    q = b.var(Var(CONF, "q0", const=True, value=Q_HOME.copy()))
    p0s = [b.var(Var(PLACEMENT, f"p0_{o.name}", const=True, value=o.init_pose.copy(), obj=i))
           for i, o in enumerate(objs)]
    for i in range(n_pieces):
        q, _ = b.pick_place(i, p0s[i], 0, q, objs[i].name, knots=knots)
    return _spec(name, objs, obbs, surfs, b, list(range(n_pieces)) if goal else [], n, steps)


def config_tetris4(n=32768, steps=100, goal=True):
    """Config 3: Tetris packing of 4 pieces {I, L, O, J} (they tile 4x4 cells) + obj_dist goal (lambda 0.25)."""
    return _tetris(4, ["I", "L", "O", "J"], (4, 4), n, steps, goal, 0, "tetris4_goal" if goal else "tetris4")


def config_tetris6_knots(n=131072, steps=100):
    """Config 4: 6 pieces {I, L, O, J, I, I} (tile 6x4 cells), 3 free knots on every motion (Fig. 9)."""
    return _tetris(6, ["I", "L", "O", "J", "I", "I"], (6, 4), n, steps, False, 3, "tetris6_knots")


def _button(name, x, y):
    """4x4x2 cm button on the table: an OBB plus its top face as a press surface (support = the button)."""
    return OBB(np.array([x, y, 0.01]), 0.0, np.array([0.02, 0.02, 0.01]), name)


def fingertip():
    """Virtual object of PressButton: the point of the closed gripper that touches the button.
    One 5 mm sphere on its frame origin (its bottom, L15); the TCP sits on that point, approach down
    (top-down grasp with no offset).  It has no constant initial placement, so it is never in the scene."""
    return Obj(name="fingertip", spheres=np.array([[0.0, 0.0, 0.005, 0.005]]), init_pose=np.zeros(4),
               footprint=0.005, grasp_xy=0.0, grasp_z=0.0)


def stick(name, length, pose):
    """Stick tool: 8 spheres of 1.5 cm along its x axis; top-down grasps anywhere along it."""
    r = 0.015
    xs = np.linspace(-length / 2 + r, length / 2 - r, 8)
    return Obj(name=name, spheres=np.array([[x, 0.0, r, r] for x in xs]), init_pose=np.array(pose, float),
               footprint=length / 2, grasp_xy=length / 2 - 0.03, grasp_y=0.003, grasp_z=0.02)


def config_stickbutton(n=4096, steps=100, direct_blue=False):
    """Stick Button (Fig. 12): press the red button directly, then pick the stick and press the
    blue button with it; the blue button sits beyond the arm's reach at the end of a walled corridor.
    direct_blue=True gives the infeasible skeleton that presses blue with the fingertip."""
    red_xy, blue_xy = (0.45, -0.25), (1.02, 0.20)
    wall_h = 0.08
    obbs = [TABLE, _button("btn_red", *red_xy), _button("btn_blue", *blue_xy),
            OBB(np.array([blue_xy[0] - 0.05, blue_xy[1] + 0.06, wall_h / 2]), 0.0, np.array([0.12, 0.01, wall_h / 2]), "wall_n"),
            OBB(np.array([blue_xy[0] - 0.05, blue_xy[1] - 0.06, wall_h / 2]), 0.0, np.array([0.12, 0.01, wall_h / 2]), "wall_s")]
    objs = [stick("stick", 0.40, [0.40, 0.15, 0.0, 0.0]), fingertip()]
    surfs = [Surface("red_top", np.array([red_xy[0], red_xy[1], 0.02, 0.0]), np.array([-0.02, -0.02]),
                     np.array([0.02, 0.02]), support_obb=1),
             Surface("blue_top", np.array([blue_xy[0], blue_xy[1], 0.02, 0.0]), np.array([-0.02, -0.02]),
                     np.array([0.02, 0.02]), support_obb=2)]
    lo, hi = _table_bounds()
    b = _Builder()
    q0 = b.var(Var(CONF, "q0", const=True, value=Q_HOME.copy()))
    p0 = b.var(Var(PLACEMENT, "p0_stick", const=True, value=objs[0].init_pose.copy(), obj=0))
    gf = b.var(Var(GRASP, "g_fingertip", obj=1))
    pr = b.var(Var(PLACEMENT, "press_red", obj=1, surface=0, lo=lo, hi=hi))
    qr = b.var(Var(CONF, "q_press_red"))
    b.actions.append(Action(MOVE_FREE, q1=q0, q2=qr))
    b.actions.append(Action(PRESS, obj=1, grasp=gf, placement=pr, surface=0, q1=qr))
    if direct_blue:
        pb = b.var(Var(PLACEMENT, "press_blue", obj=1, surface=1, lo=lo, hi=hi))
        qb = b.var(Var(CONF, "q_press_blue"))
        b.actions.append(Action(MOVE_FREE, q1=qr, q2=qb))
        b.actions.append(Action(PRESS, obj=1, grasp=gf, placement=pb, surface=1, q1=qb))
    else:
        g = b.var(Var(GRASP, "g_stick", obj=0))
        qp = b.var(Var(CONF, "q_pick_stick"))
        pb = b.var(Var(PLACEMENT, "press_blue_stick", obj=0, surface=1, lo=lo, hi=hi))
        qb = b.var(Var(CONF, "q_press_blue"))
        b.actions.append(Action(MOVE_FREE, q1=qr, q2=qp))
        b.actions.append(Action(PICK, obj=0, grasp=g, placement=p0, q1=qp))
        b.actions.append(Action(MOVE_HOLD, obj=0, grasp=g, q1=qp, q2=qb))
        b.actions.append(Action(PRESS_STICK, obj=0, grasp=g, placement=pb, surface=1, q1=qb))
    return _spec("stickbutton_direct" if direct_blue else "stickbutton", objs, obbs, surfs, b, [], n, steps)


CONFIG_NAMES = {1: "pickplace", 2: "obstruction", 3: "tetris4_goal", 4: "tetris6_knots", 5: "tetris4",
                6: "stickbutton", 7: "stickbutton_direct"}
CONFIG_SIZES = {1: 256, 2: 8192, 3: 32768, 4: 131072, 5: 1 << 20, 6: 4096, 7: 4096}


def _f32(obj):
    """Round every float constant to the nearest float32 (in place; ints/bools untouched).

    The CUDA path receives the problem in float32; rounding the shared spec once makes the oracle
    (float64 arithmetic) and the kernels (float32) solve exactly the same problem instance.
    """
    if isinstance(obj, list):
        return [_f32(o) for o in obj]
    if isinstance(obj, dict):
        return {k: _f32(v) for k, v in obj.items()}
    if isinstance(obj, np.ndarray):
        return obj.astype(np.float32).astype(np.float64) if obj.dtype.kind == "f" else obj
    if isinstance(obj, float):
        return float(np.float32(obj))
    if dataclasses.is_dataclass(obj):
        for f in dataclasses.fields(obj):
            setattr(obj, f.name, _f32(getattr(obj, f.name)))
        return obj
    return obj


def make_config(cfg: int, n: Optional[int] = None, steps: int = 100) -> ProblemSpec:
    """ProblemSpec of BASELINE.json config `cfg` (1-5; 6/7 = Stick Button skeletons) with all float
    constants float32-representable."""
    n = CONFIG_SIZES[cfg] if n is None else n
    if cfg == 1:
        spec = config_pickplace(n, steps)
    elif cfg == 2:
        spec = config_obstruction(n, steps)
    elif cfg == 3:
        spec = config_tetris4(n, steps, goal=True)
    elif cfg == 4:
        spec = config_tetris6_knots(n, steps)
    elif cfg == 5:
        spec = config_tetris4(n, steps, goal=False)
    elif cfg in (6, 7):   # Stick Button family (not a BASELINE config: parity / planner only)
        spec = config_stickbutton(n, steps, direct_blue=cfg == 7)
    else:
        raise ValueError(cfg)
    return _f32(spec)
